python tools/step_once.py --config 5 --steps 1 > gpurun_out/r2f_step5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_t3 -c 1 -o gpurun_out/r2f_k_t3_c5 \
  python tools/step_once.py --config 5 --steps 1 > gpurun_out/r2f_ncu5.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/r2f_ncu5.log
