for ur in 0 256 1024 4096; do echo "== LG_ULTRA_ROWS=$ur"; LG_ULTRA_ROWS=$ur timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee -a gpurun_out/r02bg_ultra.txt; done
