# warp-block SpMV: kernel tests + A/B timing against the round-1 kernel
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/r02b_kernels.log 2>&1; echo "kernel tests rc=$?"
tail -15 gpurun_out/r02b_kernels.log
timeout 600 python scripts/spmv_ab.py C2 C3 C4 C5 > gpurun_out/r02b_ab_new.jsonl 2>&1; echo "ab new rc=$?"
LG_LIB_OVERRIDE=build/variants/old.so timeout 600 python scripts/spmv_ab.py C3 C4 C5 > gpurun_out/r02b_ab_old.jsonl 2>&1; echo "ab old rc=$?"
cat gpurun_out/r02b_ab_new.jsonl gpurun_out/r02b_ab_old.jsonl
