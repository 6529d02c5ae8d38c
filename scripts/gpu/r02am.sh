# round-2 final evidence: GPU suite, smoke, bench lines (C4 headline with the live gather floor, C5, reference arm),
# launch list + full ncu capture of the SpMV
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02am_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02am_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02am_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02am_smoke.log
timeout 1500 python bench.py > gpurun_out/r02am_bench.json 2> gpurun_out/r02am_bench.err; echo "bench rc=$?"; head -c 1800 gpurun_out/r02am_bench.json
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/r02am_bench_c5.json 2> gpurun_out/r02am_bench_c5.err; echo "bench c5 rc=$?"; head -c 2500 gpurun_out/r02am_bench_c5.json
timeout 600 python bench.py --impl reference > gpurun_out/r02am_reference.json 2>&1; echo "reference rc=$?"; tail -c 600 gpurun_out/r02am_reference.json
