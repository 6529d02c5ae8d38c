# cluster-sweep micro (per-level cost of a one-cluster level-synchronous sweep) and
# the SpMV deferred-finish variants
./scripts/micro/sweepchain > gpurun_out/r02af_sweepchain.txt 2>&1; cat gpurun_out/r02af_sweepchain.txt
./scripts/micro/cluster > gpurun_out/r02af_cluster.txt 2>&1; tail -40 gpurun_out/r02af_cluster.txt
for v in base defer defer3; do
  if [ $v = base ]; then unset LG_LIB_OVERRIDE; else export LG_LIB_OVERRIDE=build/variants/$v.so; fi
  timeout 600 python scripts/spmv_ab.py C2 C3 C4 C5 > gpurun_out/r02af_$v.jsonl 2>&1
  echo "$v: $(python -c "
import json
for l in open('gpurun_out/r02af_$v.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), d.get('max_rel_err', d.get('max_abs_L1')), end='  ')
    except Exception: pass
")"
done
