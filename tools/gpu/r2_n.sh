for d in 2 3 6 12; do for N in 1 8; do
  t=""; for r in 0 3; do t="$t $(BBF_UNIT_DIV=$d BBF_FAKE_WORLD=$r/$N BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 5 --steps 3 2>&1 | grep -E "engine" | tail -1 | cut -c15-30)"; done; echo "div $d N=$N ranks 0,3: $t"
done; done
