timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -k "full_per_vertex or zoned or sweep or kmn or config or corpus or topk or per_edge" 2>&1 | tail -2
bash tools/gpu/ab.sh "epiold default"
