timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 4 --steps 3 --path dense 2>&1 | grep -E "dense:|count " | tail -2 | cut -c1-160
BBF_DENSE_F4_TP=1 BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 4 --steps 3 --path dense 2>&1 | grep -E "dense:|count " | tail -2 | cut -c1-160
