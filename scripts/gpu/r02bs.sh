for g in 2 4 5; do echo "== GATE=$g"; LG_SWEEP_GATE=$g timeout 600 python scripts/ic0_time.py C2 C3 C4 2>&1 | tee -a gpurun_out/r02bs_gate.txt; done
for tt in 64 256; do echo "== TASK_TARGET=$tt"; LG_TASK_TARGET=$tt timeout 600 python scripts/ic0_time.py C2 C3 C4 2>&1 | tee -a gpurun_out/r02bs_gate.txt; done
