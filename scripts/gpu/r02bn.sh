# L2 prefetch of the sweep head's structure at kernel start
for k in 0 1; do echo "== LG_IC0_NOHEADPF=$k"; if [ $k = 1 ]; then export LG_IC0_NOHEADPF=1; fi; timeout 600 python scripts/ic0_time.py C3 C4 2>&1 | tee -a gpurun_out/r02bn_headpf.txt; done
unset LG_IC0_NOHEADPF
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "ic0" > gpurun_out/r02bn_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02bn_tests.log
