for ml in 8 32; do echo "== SPLITMIN=12 MERGELEN=$ml"; LG_IC0_SPLITMIN=12 LG_IC0_MERGELEN=$ml timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bo_mergeparams.txt; done
echo "== SPLITMIN=12 MERGELEN=16 (repeat)"; LG_IC0_SPLITMIN=12 timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bo_mergeparams.txt
