# level-merged IC(0) sweeps (2 passes, default): full GPU suite, smoke; worker-warp count variants
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02ar_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r02ar_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02ar_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02ar_smoke.log
for v in flow448 flow512; do
  echo "== $v"; LG_LIB_OVERRIDE=build/variants/$v.so timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02ar_threads.txt
done
