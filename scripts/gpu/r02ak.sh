# dataflow sweep: one poll per warp on the deepest missing input (default) vs one per lane (probe1 variant)
LG_SWEEP_CTA=0 timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "ic0" > gpurun_out/r02ak_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r02ak_tests.log
LG_SWEEP_CTA=0 timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 > gpurun_out/r02ak_new.txt 2>&1; cat gpurun_out/r02ak_new.txt
LG_SWEEP_CTA=0 LG_LIB_OVERRIDE=build/variants/probe1.so timeout 600 python scripts/ic0_time.py C1 C2 C3 C4 > gpurun_out/r02ak_probe1.txt 2>&1; cat gpurun_out/r02ak_probe1.txt
LG_SWEEP_CTA=0 timeout 300 python scripts/flow_trace.py C4 > gpurun_out/r02ak_trace_c4.txt 2>&1; cat gpurun_out/r02ak_trace_c4.txt
