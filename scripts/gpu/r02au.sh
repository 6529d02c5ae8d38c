# hub rows: deepest inputs first (late inputs in chunk 0): apply times and IC(0) tests, with and without
timeout 300 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee gpurun_out/r02au_hubsort.txt
LG_IC0_NOHUBSORT=1 timeout 300 python scripts/ic0_time.py C1 C2 C3 C4 2>&1 | tee gpurun_out/r02au_nohubsort.txt
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "ic0" > gpurun_out/r02au_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r02au_tests.log
LG_IC0_MERGE=2 timeout 300 python scripts/flow_trace.py C4 2>&1 | tee gpurun_out/r02au_trace_c4.txt
