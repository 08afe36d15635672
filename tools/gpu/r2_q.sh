for rep in 1 2; do for v in prev default; do
  if [ "$v" = default ]; then L=paper_2308_07932_b200/libbbf.so; else L=paper_2308_07932_b200/_build_$v/libbbf.so; fi
  BBF_LIB=$L python bench.py --no-cpu-baseline --steps 10 --e2e-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,1), round(d['ms_per_step'],2), round(d['count_only']['ms_per_step'],2), round(d['roofline']['ms_per_launch'],2))"
done; done
