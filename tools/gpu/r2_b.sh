# Round 2, second call: whole GPU suite (new collective / top-k / estimate / gloo tests), smoke.
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r2b_pytest.log 2>&1; echo "gpu suite rc=$?"
tail -5 gpurun_out/r2b_pytest.log
timeout 300 python -c "import __graft_entry__ as e; e.build(); e.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2b_smoke.log
