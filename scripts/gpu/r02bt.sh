# round-2 final: GPU suite, smoke, bench lines (C4, C5, reference arm), launch list, IC(0) apply times
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02k_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r02k_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02k_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02k_smoke.log
timeout 300 python scripts/ic0_time.py C1 C2 C3 C4 > gpurun_out/r02k_ic0_time.txt 2>&1; cat gpurun_out/r02k_ic0_time.txt
timeout 1500 python bench.py > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; echo "bench rc=$?"; head -c 300 gpurun_out/r02k_bench.json
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/r02k_bench_c5.json 2> gpurun_out/r02k_bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r02k_reference.json 2>&1; echo "reference rc=$?"
python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02k_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02k_ncu1.log 2>&1; echo "launches rc=$?"
timeout 300 python scripts/dacg_iter.py C4 > gpurun_out/r02k_dacg_iter_c4.txt 2>&1; cat gpurun_out/r02k_dacg_iter_c4.txt
timeout 600 python scripts/iter_roofline.py C4 > gpurun_out/r02k_iter_roofline_ic0.json 2> gpurun_out/r02k_iter_roofline_ic0.err; echo "iter roofline rc=$?"
