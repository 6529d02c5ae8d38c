# deferred long-row finish: tests + A/B (defer on / off) on C3 C4 C5; C1/C2 IC(0) apply per sweep mode
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/r02s_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02s_tests.log
for d in 1 0; do
  LG_SPMV_DEFER=$d timeout 300 python scripts/spmv_ab.py C3 C4 C5 > gpurun_out/r02s_defer$d.jsonl 2>&1; echo "defer=$d: $(python -c "
import json
for l in open('gpurun_out/r02s_defer$d.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), end='  ')
    except Exception: pass
")"
done
LG_SPMV_DEFER=1 LG_SPMV_PANELS=0 timeout 300 python scripts/spmv_ab.py C5 > gpurun_out/r02s_c5np.jsonl 2>&1; echo "defer=1 nopanels: $(tail -1 gpurun_out/r02s_c5np.jsonl)"
for m in 1 0; do LG_SWEEP_MODE=$m timeout 300 python scripts/ic0_time.py C1 C2 > gpurun_out/r02s_ic0_m$m.txt 2>&1; echo "sweep mode $m: $(cat gpurun_out/r02s_ic0_m$m.txt | tr '\n' ' ')"; done
