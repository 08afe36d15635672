python tools/step_once.py --config 3 --steps 1 > gpurun_out/p4_step3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/p4_k_t3_c3 \
  python tools/step_once.py --config 3 --steps 1 > gpurun_out/p4_ncu3.log 2>&1
tail -1 gpurun_out/p4_ncu3.log
