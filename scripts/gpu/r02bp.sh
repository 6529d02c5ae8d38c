for sm in 12 16 32; do echo "== SPLITMIN=$sm"; LG_IC0_SPLITMIN=$sm timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bo_mergeparams.txt; done
