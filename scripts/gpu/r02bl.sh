# final check of the shipped library: GPU suite, smoke, one default bench line
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02i_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02i_tests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02i_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02i_smoke.log
timeout 1500 python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo "bench rc=$?"; head -c 400 gpurun_out/r02i_bench.json
