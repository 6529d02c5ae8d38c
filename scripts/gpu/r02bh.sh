for tt in 0 128 512 2048; do echo "== LG_TASK_TARGET=$tt"; LG_TASK_TARGET=$tt timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bh_tasktarget.txt; done
