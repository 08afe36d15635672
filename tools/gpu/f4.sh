timeout 600 python -m pytest tests -m gpu -x -q -k "dense or kmn or complete or config4 or fake" 2>&1 | tail -3
BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 4 --steps 3 --path dense 2>&1 | grep -E "dense:|count " | tail -2
BBF_DENSE_I8=1 BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 4 --steps 3 --path dense 2>&1 | grep -E "dense:|count " | tail -2
