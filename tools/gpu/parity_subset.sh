# Full-size parity subset (per-vertex configs 3-5 and the zoned graph, sweep, top-k, shards) for the
# default library or a variant.  Usage: bash tools/gpu/parity_subset.sh [VARIANT]
L=paper_2308_07932_b200/libbbf.so
[ -n "$1" ] && L=paper_2308_07932_b200/_build_$1/libbbf.so
BBF_LIB=$L timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q \
  -k "full_per_vertex or zoned or sweep or topk or pairs or fake_world" 2>&1 | tail -1
