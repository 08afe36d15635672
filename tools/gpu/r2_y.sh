# T2 tier bound (env BBF_T2_MAX): hash tier vs hub windows for mid-size starts
for v in 8192 10240 12288; do for c in 5 3; do echo "== t2max=$v c$c: $(BBF_T2_MAX=$v BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 3 2>&1 | grep -E "engine|count" | tail -2 | cut -c1-90 | tr '\n' ' ')"; done; done
