# ncu launch list of the bench command + one full capture of the hub kernel (config 5 and 3)
python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/p_bench5.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/p_launches_c5.csv \
  python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/p_ncu_launch.log 2>&1
python tools/step_once.py --config 5 --steps 1 > gpurun_out/p_step5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/p_k_t3_c5 \
  python tools/step_once.py --config 5 --steps 1 > gpurun_out/p_ncu_full5.log 2>&1
python tools/step_once.py --config 3 --steps 1 > gpurun_out/p_step3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/p_k_t3_c3 \
  python tools/step_once.py --config 3 --steps 1 > gpurun_out/p_ncu_full3.log 2>&1
ls -la gpurun_out
