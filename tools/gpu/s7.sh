cp tools/gpu/libs/libbbf_prof.so paper_2308_07932_b200/libbbf.so; BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 5 --steps 2 2>&1 | grep -E "engine|phases" | tail -2 | cut -c1-150
cp tools/gpu/libs/libbbf_plain.so paper_2308_07932_b200/libbbf.so
bash tools/gpu/t2.sh
