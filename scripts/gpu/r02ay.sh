# resident vs dataflow sweeps on the level-merged schedules
for th in 512 256; do LG_SWEEP_CTA_THREADS=$th timeout 300 python scripts/ic0_modes.py C1 C2 2>&1 | tee -a gpurun_out/r02ay_modes.jsonl; done
for m in 3 4; do LG_IC0_MERGE=$m LG_SWEEP_CTA_THREADS=512 timeout 300 python scripts/ic0_modes.py C1 C2 2>&1 | tee -a gpurun_out/r02ay_modes.jsonl; done
