# level-merged IC(0) sweeps: depth, entries, apply time and error against the oracle for 0-3 merge passes; IC(0) tests
for m in 0 1 2 3; do
  echo "== LG_IC0_MERGE=$m"; LG_IC0_MERGE=$m timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02an_merge.txt
done
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "ic0" > gpurun_out/r02an_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r02an_tests.log
