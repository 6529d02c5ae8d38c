# full GPU suite, bench line, launch list and ncu capture of the SpMV
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02r_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02r_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02r_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02r_smoke.log
timeout 1200 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err; echo "bench rc=$?"; tail -c 300 gpurun_out/r02r_bench.json
python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02r_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02r_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02r_ncu1.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:wspmv -s 3 -c 1 -o gpurun_out/r02r_spmv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02r_ncu2.log 2>&1; echo "ncu full rc=$?"
