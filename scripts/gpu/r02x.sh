# reference IC(0) ladder on device-built R-MAT (C5 family)
free -g | head -2; nproc
for s in 20 22; do timeout 900 python scripts/ic0_ladder.py $s --solve > gpurun_out/r02x_ic0_s$s.jsonl 2> gpurun_out/r02x_ic0_s$s.err; echo "scale $s rc=$?"; tail -1 gpurun_out/r02x_ic0_s$s.jsonl; tail -2 gpurun_out/r02x_ic0_s$s.err; done
timeout 1200 python scripts/ic0_ladder.py 24 > gpurun_out/r02x_ic0_s24.jsonl 2> gpurun_out/r02x_ic0_s24.err; echo "scale 24 rc=$?"; tail -1 gpurun_out/r02x_ic0_s24.jsonl; tail -2 gpurun_out/r02x_ic0_s24.err
