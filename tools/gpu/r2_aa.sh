# static first batches / records / middle batches (variant st) vs default: parity subset + timing
timeout 900 env BBF_LIB=paper_2308_07932_b200/_build_st/libbbf.so python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -k "full_per_vertex or zoned or sweep or fake_world" 2>&1 | tail -1
bash tools/gpu/ab.sh "default st"
