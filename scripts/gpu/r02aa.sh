# warp-specialised SpMV (LG_SPMV_WS=1): tests + A/B of gather/reduce warp splits
LG_SPMV_WS=1 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "spmv or row_part or laplacian or panel or export" > gpurun_out/r02aa_tests.log 2>&1; echo "ws tests rc=$?"; tail -2 gpurun_out/r02aa_tests.log
for v in ws24_8 ws20_12 ws16_16 ws12_20; do LG_SPMV_WS=1 LG_LIB_OVERRIDE=build/variants/$v.so timeout 300 python scripts/spmv_ab.py C2 C3 C4 C5 > gpurun_out/r02aa_$v.jsonl 2>&1; echo "$v: $(python -c "
import json
for l in open('gpurun_out/r02aa_$v.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), end='  ')
    except Exception: pass
")"; done
timeout 300 python scripts/spmv_ab.py C2 C3 C4 C5 > gpurun_out/r02aa_base.jsonl 2>&1; echo "base: $(python -c "
import json
for l in open('gpurun_out/r02aa_base.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), end='  ')
    except Exception: pass
")"
