LG_SWEEP_CTA=1 timeout 300 python scripts/flow_trace.py C1 --levels > gpurun_out/r02ah_trace_c1.txt 2>&1; head -70 gpurun_out/r02ah_trace_c1.txt
LG_SWEEP_CTA=1 timeout 300 python scripts/flow_trace.py C2 > gpurun_out/r02ah_trace_c2.txt 2>&1; cat gpurun_out/r02ah_trace_c2.txt
