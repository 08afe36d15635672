for c in 5 3; do BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 3 2>&1 | grep -E "engine" | tail -1 | cut -c1-60; done
