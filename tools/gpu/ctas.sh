# hub-kernel geometry variants: CTAs per SM x threads (window shrinks with CTAs per SM)
for v in "-DBBF_T3_CTAS=1 -DBBF_T3_THREADS=1024" "-DBBF_T3_CTAS=2 -DBBF_T3_THREADS=512" "-DBBF_T3_CTAS=1 -DBBF_T3_THREADS=768"; do
  BBF_NVCC_EXTRA="$v" python -m paper_2308_07932_b200.build --force > /dev/null 2>gpurun_out/ctas_build.err || { echo "$v build failed"; tail -3 gpurun_out/ctas_build.err; continue; }
  for c in 5 3; do
    r=$(python tools/step_once.py --config $c --steps 3 2>&1 | tail -1 | grep -o "device [0-9.]*, main [0-9.]*")
    echo "$v config $c: $r"
  done
done
