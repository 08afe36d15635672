for b in 20 24 28 32; do echo "bsz $b c5 $(BBF_T3_BSZ=$b BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 5 --steps 3 2>&1 | grep engine | tail -1 | cut -c1-30)"; done
for b in 8 10 12; do echo "bsz $b c3 $(BBF_T3_BSZ=$b BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 3 --steps 3 2>&1 | grep engine | tail -1 | cut -c1-30)"; done
