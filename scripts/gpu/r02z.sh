# C5 (R-MAT 26) with the reference IC(0): host factor (level-parallel), sweeps, DACG 5 pairs next to FSAI
timeout 5400 python scripts/ic0_ladder.py 26 --solve > gpurun_out/r02z_ic0_s26.jsonl 2> gpurun_out/r02z_ic0_s26.err; echo "scale 26 rc=$?"; tail -1 gpurun_out/r02z_ic0_s26.jsonl; tail -3 gpurun_out/r02z_ic0_s26.err
