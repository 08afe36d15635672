for c in 3 5; do BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 1 2>&1 | grep -E "engine|phases|epilogue" | cut -c1-200; done
