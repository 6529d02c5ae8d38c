# polling variants on the merged schedule
for v in spinall poll2 rcp; do echo "== $v"; LG_LIB_OVERRIDE=build/variants/$v.so timeout 600 python scripts/ic0_time.py C2 C3 C4 2>&1 | tee -a gpurun_out/r02ax_poll.txt; done
