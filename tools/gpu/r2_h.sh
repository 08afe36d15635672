for v in prof pNOATOM pNOLDS pNOEPI; do for c in 5; do echo "== $v c$c: $(BBF_LIB=paper_2308_07932_b200/_build_$v/libbbf.so BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 2 2>&1 | grep -E "phases|engine" | tail -2 | cut -c1-140 | tr '\n' ' ')"; done; done
bash tools/gpu/ab.sh "xNOATOM xNOLDS xNOEPI xall"
