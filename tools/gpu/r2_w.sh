# A/B: window-uniform half-field width in the long-record pass 2 (variant uh) vs the default build
timeout 600 env BBF_LIB=paper_2308_07932_b200/_build_uh/libbbf.so python -m pytest tests/test_gpu_fullsize.py -x -q -k "full_per_vertex and (config3 or zoned)" 2>&1 | tail -1
bash tools/gpu/ab.sh "default uh"
