# level-merged sweeps: gate / wide-level knobs
for m in 1 2; do for g in 2 3 4 6; do
  echo "== MERGE=$m GATE=$g"; LG_IC0_MERGE=$m LG_SWEEP_GATE=$g timeout 600 python scripts/ic0_time.py C3 C4 2>&1 | tee -a gpurun_out/r02aq_knobs.txt
done; done
for w in 4096 65536; do
  echo "== MERGE=2 WIDE_ROWS=$w"; LG_IC0_MERGE=2 LG_WIDE_ROWS=$w timeout 600 python scripts/ic0_time.py C3 C4 2>&1 | tee -a gpurun_out/r02aq_knobs.txt
done
LG_IC0_MERGE=2 timeout 300 python scripts/flow_trace.py C4 2>&1 | tee gpurun_out/r02aq_trace_c4.txt
