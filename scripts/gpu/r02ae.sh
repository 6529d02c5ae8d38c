# re-entry check of the restored tree: GPU suite, smoke, bench line
set -x
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02ae_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02ae_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02ae_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02ae_smoke.log
timeout 1500 python bench.py > gpurun_out/r02ae_bench.json 2> gpurun_out/r02ae_bench.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r02ae_bench.json
timeout 300 python scripts/ic0_time.py C1 C2 C3 C4 > gpurun_out/r02ae_ic0_time.txt 2>&1; cat gpurun_out/r02ae_ic0_time.txt
