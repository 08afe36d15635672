python tools/step_once.py --config 5 --steps 1 > gpurun_out/p5_step5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/p5_k_t3_c5 \
  python tools/step_once.py --config 5 --steps 1 > gpurun_out/p5_ncu5.log 2>&1
tail -2 gpurun_out/p5_ncu5.log
