timeout 300 python scripts/flow_trace.py C4 --levels 2>&1 | tee gpurun_out/r02bm_trace_levels_c4.txt | head -30
