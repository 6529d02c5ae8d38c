# merge passes with the hub ordering and the wide CTA in place
for m in 2 3 4; do echo "== LG_IC0_MERGE=$m"; LG_IC0_MERGE=$m timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02aw_merge.txt; done
