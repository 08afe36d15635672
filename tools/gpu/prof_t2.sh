python tools/step_once.py --config 3 --steps 1 > gpurun_out/pt2_step5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_t[12] -c 5 -o gpurun_out/pt2_k_t2_c5 \
  python tools/step_once.py --config 3 --steps 1 > gpurun_out/pt2_ncu5.log 2>&1
tail -2 gpurun_out/pt2_ncu5.log
