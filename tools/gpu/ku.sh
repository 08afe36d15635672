# compile-time hub-kernel variants (steps per iteration kU, entries per chunk kCE): count device ms
for v in "-DBBF_T3_KU=2" "-DBBF_T3_KU=3" "-DBBF_T3_KU=1" "-DBBF_T3_CE=16" "-DBBF_T3_CE=4"; do
  BBF_NVCC_EXTRA="$v" python -m paper_2308_07932_b200.build --force > /dev/null 2>gpurun_out/ku_build.err || { echo "$v build failed"; tail -3 gpurun_out/ku_build.err; continue; }
  for c in 5 3; do
    r=$(python tools/step_once.py --config $c --steps 3 2>&1 | tail -1 | grep -o "device [0-9.]*, main [0-9.]*")
    echo "$v config $c: $r"
  done
done
