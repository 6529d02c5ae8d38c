# wide schedules: entries staged through shared memory (23 worker warps, 80 registers) vs registers (15 warps)
for k in 2 1 0; do echo "== LG_FLOW_WIDE=$k"; LG_FLOW_WIDE=$k timeout 600 python scripts/ic0_time.py C3 C4 2>&1 | tee -a gpurun_out/r02bk_wide.txt; done
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "ic0" > gpurun_out/r02bk_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02bk_tests.log
