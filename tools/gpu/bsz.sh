# BBF_T3_BSZ A/B on config ${CFG:-5} (count device ms, alternating runs)
for i in 1 2 3; do for b in 16 24 32; do
  r=$(BBF_T3_BSZ=$b python tools/step_once.py --config ${CFG:-5} --steps 3 2>&1 | tail -1 | grep -o "device [0-9.]*, main [0-9.]*")
  echo "bsz $b: $r"; done; done
