# Round-1 evidence: ncu launch list of the default bench command, and one --set full capture of
# each main kernel (k_t3 on configs 5 and 3, k_dense_pair on config 4), each after a plain run.
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pr_bench5.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/pr_launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/pr_ncu_launch.log 2>&1
python tools/step_once.py --config 5 --steps 1 > gpurun_out/pr_step5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/pr_k_t3_c5 \
  python tools/step_once.py --config 5 --steps 1 > gpurun_out/pr_ncu5.log 2>&1
python tools/step_once.py --config 3 --steps 1 > gpurun_out/pr_step3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/pr_k_t3_c3 \
  python tools/step_once.py --config 3 --steps 1 > gpurun_out/pr_ncu3.log 2>&1
python tools/step_once.py --config 4 --steps 1 --path dense > gpurun_out/pr_step4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_dense_f4 -c 1 -o gpurun_out/pr_k_dense_f4q_c4 \
  python tools/step_once.py --config 4 --steps 1 --path dense > gpurun_out/pr_ncu4.log 2>&1
ls -la gpurun_out | grep pr_
