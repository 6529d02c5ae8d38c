# round-2 evidence: GPU suite, smoke, bench lines (C4 headline, C5, reference arm),
# launch list + ncu of the SpMV, C5 product DRAM traffic, scaling projection
set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02ab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02ab_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02ab_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02ab_smoke.log
timeout 1500 python bench.py > gpurun_out/r02ab_bench.json 2> gpurun_out/r02ab_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/r02ab_bench_c5.json 2> gpurun_out/r02ab_bench_c5.err; echo "bench c5 rc=$?"; tail -c 400 gpurun_out/r02ab_bench_c5.json
timeout 600 python bench.py --impl reference > gpurun_out/r02ab_reference.json 2>&1; echo "reference rc=$?"; tail -c 300 gpurun_out/r02ab_reference.json
python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02ab_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ab_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02ab_ncu1.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:wspmv -s 3 -c 1 -o gpurun_out/r02ab_spmv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02ab_ncu2.log 2>&1; echo "ncu full rc=$?"
python scripts/spmv_ab.py C5 > gpurun_out/r02ab_c5plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none \
  -k regex:"wspmv|long_finish|diag_init" -s 45 -c 9 --csv --log-file gpurun_out/r02ab_c5_traffic.csv \
  python scripts/spmv_ab.py C5 > gpurun_out/r02ab_ncu3.log 2>&1; echo "c5 traffic rc=$?"
timeout 900 python scripts/scaling_projection.py C4 --device-collectives > gpurun_out/r02ab_proj_c4.jsonl 2>&1; echo "proj c4 rc=$?"
timeout 1500 python scripts/scaling_projection.py C5 --jacobi --device-collectives > gpurun_out/r02ab_proj_c5.jsonl 2>&1; echo "proj c5 rc=$?"
