timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in 4 3; do BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 3 2>&1 | grep -E "load|dense:|engine" | tail -2 | cut -c1-180; done
