for p in dense sparse; do BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 4 --steps 3 --path $p > gpurun_out/d2_step4_$p.log 2>&1; done
BBF_DEBUG=1 timeout 300 python tools/step_once.py --config 4 --steps 2 --path dense --global-only > gpurun_out/d2_step4_dense_global.log 2>&1
tail -4 gpurun_out/d2_*.log
