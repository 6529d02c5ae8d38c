# gather microbenchmarks on C4's column stream: shared-memory hub table at full occupancy, half-warp LDGs
./scripts/micro/gather_hub2 build/data/c4_cols.bin 989777 > gpurun_out/r02al_gather_hub2.txt 2>&1; cat gpurun_out/r02al_gather_hub2.txt
