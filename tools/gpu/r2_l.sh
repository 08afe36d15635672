bash tools/gpu/ab.sh "default lm128 lm512"
for d in 1 4; do echo "dense_div $d: $(BBF_DENSE_DIV=$d BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 5 --steps 3 2>&1 | grep -E "engine" | tail -1 | cut -c1-60)"; done
