# A/B of library variants on the hub kernel: tools/gpu/ab.sh "name1 name2 ..." (default = in-tree lib)
for rep in 1 2; do
for v in $1; do
  if [ "$v" = default ]; then L=paper_2308_07932_b200/libbbf.so; else L=paper_2308_07932_b200/_build_$v/libbbf.so; fi
  for c in 5 3; do echo "== $v c$c: $(BBF_LIB=$L BBF_DEBUG=1 timeout 300 python tools/step_once.py --config $c --steps 3 2>&1 | grep -E "engine" | tail -1 | cut -c1-60)"; done
done; done
