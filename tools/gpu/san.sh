timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 3 5; do BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 2 2>&1 | grep -E "load" | tail -1 | cut -c1-60; done
# memcheck + racecheck of the hub kernel path on a small graph (config 2) and the dense path (config 1)
cat > /tmp/san_run.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2308_07932_b200 import bbf
from synth import graphs as G
for g, fl in ((G.config2(), bbf.BBF_FORCE_SPARSE), (G.config1(), bbf.BBF_FORCE_DENSE)):
    with bbf.Graph.from_synth(g, flags=fl) as h:
        print(h.count_global()["balanced"], h.count_per_vertex()[0]["balanced"], h.count_pairs_topk(5))
PY
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/san_run.py > gpurun_out/san_memcheck.log 2>&1; tail -4 gpurun_out/san_memcheck.log
