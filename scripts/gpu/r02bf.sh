# per-level lane classes (narrow levels: more lanes per row): thresholds
for fr in 2048 4096 1024 0; do echo "== LG_FINE_ROWS=$fr"; LG_FINE_ROWS=$fr timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bf_fine.txt; done
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "ic0" > gpurun_out/r02bf_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02bf_tests.log
