for c in 3 5; do BBF_DEBUG=2 timeout 300 python tools/step_once.py --config $c --steps 1 2>&1 | grep "work \["; done
