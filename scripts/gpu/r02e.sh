# warp SpMV + L2 prefetch of x / diag; compacted accumulating panels for C5
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/r02e_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02e_tests.log
timeout 300 python scripts/spmv_ab.py C3 C4 C5 > gpurun_out/r02e_ab_pf.jsonl 2>&1; echo "pf rc=$?"; cat gpurun_out/r02e_ab_pf.jsonl
LG_SPMV_PREFETCH=0 timeout 300 python scripts/spmv_ab.py C3 C4 > gpurun_out/r02e_ab_nopf.jsonl 2>&1; echo "nopf rc=$?"; cat gpurun_out/r02e_ab_nopf.jsonl
LG_SPMV_PANELS=0 timeout 300 python scripts/spmv_ab.py C5 > gpurun_out/r02e_ab_c5_nopanel.jsonl 2>&1; echo "c5 nopanel rc=$?"; cat gpurun_out/r02e_ab_c5_nopanel.jsonl
