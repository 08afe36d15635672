timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "full_per_vertex and (config3 or zoned)" 2>&1 | tail -1
bash tools/gpu/ab.sh "default z2 z4 z5"
