# full GPU suite on the warp SpMV + timing
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02l_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02l_tests.log
timeout 300 python scripts/spmv_ab.py C2 C3 C4 C5 > gpurun_out/r02l_ab.jsonl 2>&1; echo "ab rc=$?"; cat gpurun_out/r02l_ab.jsonl
