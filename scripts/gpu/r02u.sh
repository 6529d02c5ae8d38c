# gather-pipelined SpMV: tests on gp3 then A/B
LG_LIB_OVERRIDE=build/variants/gp3.so timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "spmv or row_part or laplacian or spmm or panel" > gpurun_out/r02u_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02u_tests.log
for v in gp3 gp2 nogp; do
  LG_LIB_OVERRIDE=build/variants/$v.so timeout 300 python scripts/spmv_ab.py C3 C4 C5 > gpurun_out/r02u_$v.jsonl 2>&1; echo "$v: $(python -c "
import json
for l in open('gpurun_out/r02u_$v.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), end='  ')
    except Exception: pass
")"
done
