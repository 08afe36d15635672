# record statistics of the hub kernel (diagnostic build): record lengths, chunk fill, pass-2 usefulness
for c in 5 3; do echo "== c$c"; BBF_LIB=paper_2308_07932_b200/_build_rs/libbbf.so BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 1 2>&1 | grep -E "t3 (records|pass-2|entries)"; done
# timing only (results wrong): the long records' entries synthesised instead of loaded (!S1 zones only)
bash tools/gpu/ab.sh "default noldg"
