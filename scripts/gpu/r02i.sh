# branch-free segmented fold: tests + timing
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/r02i_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02i_tests.log
timeout 300 python scripts/spmv_ab.py C2 C3 C4 C5 > gpurun_out/r02i_ab.jsonl 2>&1; echo "ab rc=$?"; cat gpurun_out/r02i_ab.jsonl
LG_SPMV_PANELS=0 timeout 300 python scripts/spmv_ab.py C5 > gpurun_out/r02i_ab_c5np.jsonl 2>&1; cat gpurun_out/r02i_ab_c5np.jsonl
