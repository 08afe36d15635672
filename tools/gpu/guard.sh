# BBF_GUARD=1: guard bytes around every library allocation, checked at each free (aborts on an
# out-of-bounds write); the sanitizer driver, the GPU test suite and one step of configs 3-5
export BBF_GUARD=1
timeout 900 python tests/scripts/sanitize_run.py > gpurun_out/guard_san.log 2>&1; echo "sanitize_run rc=$?"; tail -2 gpurun_out/guard_san.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/guard_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/guard_pytest.log
for c in 3 4 5 6; do timeout 600 python tools/step_once.py --config $c --steps 1 > gpurun_out/guard_step$c.log 2>&1; echo "step config $c rc=$?"; tail -2 gpurun_out/guard_step$c.log; done
timeout 600 python tools/step_once.py --config 4 --steps 1 --path sparse > gpurun_out/guard_step4s.log 2>&1; echo "step config 4 sparse rc=$?"; tail -2 gpurun_out/guard_step4s.log
