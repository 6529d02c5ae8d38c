# pipelined warp-block SpMV: A/B of occupancy variants against round 1
for v in pipe_m4 pipe_m3 old; do
  LG_LIB_OVERRIDE=build/variants/$v.so timeout 300 python scripts/spmv_ab.py C3 C4 > gpurun_out/r02d_ab_$v.jsonl 2>&1; echo "$v rc=$?"
  cat gpurun_out/r02d_ab_$v.jsonl
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "spmv or row_part or laplacian" > gpurun_out/r02d_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02d_tests.log
