# epilogue fast path for one-end-per-word zones (variant e16) vs default: parity subset + timing
timeout 900 env BBF_LIB=paper_2308_07932_b200/_build_e16/libbbf.so python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -k "full_per_vertex or zoned or sweep or topk or pairs" 2>&1 | tail -1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
bash tools/gpu/ab.sh "default e16"
