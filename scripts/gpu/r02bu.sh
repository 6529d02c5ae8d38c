for wt in 0 128 100000; do echo "== LG_FLOW_WIDE_TASKS=$wt"; LG_FLOW_WIDE_TASKS=$wt timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bu_widetasks.txt; done
