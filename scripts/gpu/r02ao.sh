# full GPU suite with the level-merged IC(0) sweeps (LG_IC0_MERGE default)
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02ao_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r02ao_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02ao_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02ao_smoke.log
