echo "== LG_LANES_ALT=2 (more lanes per row)"; LG_LANES_ALT=2 timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bd_lanes.txt
