# Hub-kernel diagnostics of a library variant (built with e.g. -DBBF_T3_PROF -DBBF_T3_WINPROF, -DBBF_T3_RECSTAT,
# -DBBF_T3_LATPROF): one step of configs 5 and 3 with BBF_DEBUG, the "[bbf] t3" lines.
# Usage: bash tools/gpu/diag.sh VARIANT   (loads paper_2308_07932_b200/_build_VARIANT/libbbf.so)
for c in 5 3; do
  echo "== $1 c$c"
  BBF_LIB=paper_2308_07932_b200/_build_$1/libbbf.so BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 1 2>&1 | grep -E "\[bbf\] (t3|engine|plan)"
done
