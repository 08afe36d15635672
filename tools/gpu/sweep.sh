# knob sweep of the sparse engine: count device ms (second step) for configs 3 and 5
for c in 3 5; do
  for kv in "" "BBF_DENSE_DIV=1" "BBF_DENSE_DIV=4" "BBF_T3_BSZ=8" "BBF_T3_BSZ=24" "BBF_T2_MAX=6144" "BBF_T2_MAX=12288"; do
    r=$(env $kv python tools/step_once.py --config $c --steps 2 2>&1 | tail -1 | grep -o "count [0-9.]* ms (device [0-9.]*, main [0-9.]*)")
    echo "config $c ${kv:-default}: $r"
  done
done
