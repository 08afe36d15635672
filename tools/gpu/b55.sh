for i in 1 2 3; do timeout 900 python bench.py --no-cpu-baseline > gpurun_out/b55_$i.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/b55_$i.json')); print(round(d['value']/1e9,1), round(d['e2e']['value']/1e9,1), round(d['e2e']['ms_per_step'],2))"; done
