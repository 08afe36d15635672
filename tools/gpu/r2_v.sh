# per-phase cycles per window-size bin and unit-size bins (diagnostic build, config 5 and 3)
for c in 5 3; do echo "== c$c"; BBF_LIB=paper_2308_07932_b200/_build_prof/libbbf.so BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 2 2>&1 | grep -E "t3 " | tail -16; done
