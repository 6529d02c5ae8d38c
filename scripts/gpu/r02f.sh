# gather floor on C4's real column stream vs shuffled / uniform / hub-staged
./scripts/micro/gather_real build/data/c4_cols.bin 989777 2>&1 | tee gpurun_out/r02f_gather_real.txt
