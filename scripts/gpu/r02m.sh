# occupancy / pipelining variants of the warp SpMV
for v in p1m4 p0m4 p0m5 p0m6 p1m3; do
  LG_LIB_OVERRIDE=build/variants/$v.so timeout 300 python scripts/spmv_ab.py C3 C4 > gpurun_out/r02m_$v.jsonl 2>&1; echo "$v: $(python -c "
import json
for l in open('gpurun_out/r02m_$v.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), end='  ')
    except Exception: pass
")"
done
