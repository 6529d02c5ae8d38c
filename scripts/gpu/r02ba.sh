# after the host-system refactor: GPU suite, smoke, apply times
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02g_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02g_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02g_smoke.log
timeout 300 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee gpurun_out/r02g_ic0_time.txt
