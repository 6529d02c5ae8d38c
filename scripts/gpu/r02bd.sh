# lanes-per-row classes on the merged schedule
for a in 0 1 2; do echo "== LG_LANES_ALT=$a"; LG_LANES_ALT=$a timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bd_lanes.txt; done
