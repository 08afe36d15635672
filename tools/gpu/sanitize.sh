# compute-sanitizer over tests/scripts/sanitize_run.py: memcheck (full), racecheck and synccheck (--quick)
CS=/usr/local/cuda/bin/compute-sanitizer
python tests/scripts/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/san_plain.log
timeout 1500 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python tests/scripts/sanitize_run.py > gpurun_out/san_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -4 gpurun_out/san_memcheck.log
timeout 1500 $CS --tool racecheck --racecheck-report hazard --error-exitcode 9 --print-limit 20 python tests/scripts/sanitize_run.py --quick > gpurun_out/san_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -4 gpurun_out/san_racecheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 --print-limit 20 python tests/scripts/sanitize_run.py --quick > gpurun_out/san_synccheck.log 2>&1; echo "synccheck rc=$?"; tail -4 gpurun_out/san_synccheck.log
