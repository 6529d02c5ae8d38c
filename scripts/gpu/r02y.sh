# (1) fold without the c[] array: A/B; (2) IC(0) per-level step on hub-free grids vs C4
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "spmv or row_part or laplacian or panel or export" > gpurun_out/r02y_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02y_tests.log
for v in head_m4 nogp; do
  LG_LIB_OVERRIDE=build/variants/$v.so timeout 300 python scripts/spmv_ab.py C3 C4 C5 > gpurun_out/r02y_$v.jsonl 2>&1; echo "$v: $(python -c "
import json
for l in open('gpurun_out/r02y_$v.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), end='  ')
    except Exception: pass
")"
done
timeout 300 python scripts/flow_trace.py grid150 grid300 grid600 > gpurun_out/r02y_flow_grid.txt 2>&1; grep -E "fwd:|bwd:" gpurun_out/r02y_flow_grid.txt
