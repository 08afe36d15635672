cp tools/gpu/libs/libbbf_prof.so paper_2308_07932_b200/libbbf.so
for c in 5 3; do BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 2 2>&1 | grep -E "engine|phases|CTA ends|epilogue" | tail -4 | cut -c1-150; done
