# integer-weight computed values: tests + timing, then flow trace of the IC(0) apply
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/r02o_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02o_tests.log
timeout 300 python scripts/spmv_ab.py C2 C3 C4 C5 > gpurun_out/r02o_ab.jsonl 2>&1; echo "ab: $(python -c "
import json
for l in open('gpurun_out/r02o_ab.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), end='  ')
    except Exception: pass
")"
timeout 300 python scripts/flow_trace.py C4 C3 > gpurun_out/r02o_flow.txt 2>&1; echo "flow rc=$?"; cat gpurun_out/r02o_flow.txt
LG_SWEEP_GATE=8 timeout 300 python scripts/flow_trace.py C4 > gpurun_out/r02o_flow_g8.txt 2>&1; cat gpurun_out/r02o_flow_g8.txt
