for m in 3 4; do echo "== LG_IC0_MERGE=$m"; LG_IC0_MERGE=$m timeout 600 python scripts/ic0_time.py C1 C2 C3 2>&1 | tee -a gpurun_out/r02bi_merge.txt; done
