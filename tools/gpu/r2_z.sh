# tiny-window latency marks (diagnostic build): when warps reach the batches, when records / chunks arrive, pass ends
for c in 5 3; do echo "== c$c"; BBF_LIB=paper_2308_07932_b200/_build_lat/libbbf.so BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 1 2>&1 | grep -E "tiny|t3 phases"; done
