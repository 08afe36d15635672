# Runtime-knob sweep of the hub kernel (env variables read by the library): k_t3 ms of configs 5 and 3.
# Usage: bash tools/gpu/knobs.sh "BBF_T3_BSZ=0 BBF_T3_BSZ=8 BBF_DENSE_DIV=4 ..."
for kv in $1; do for c in 5 3; do
  echo "== $kv c$c: $(env $kv BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 3 2>&1 | grep -E "engine" | tail -1 | cut -c1-60)"
done; done
