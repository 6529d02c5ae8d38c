# small single-CTA IC(0) sweep: tests, apply timing, C1/C2 solves (small on / off)
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solvers.py -x -q -p no:cacheprovider -k "ic0 or dacg or jd or irlm or kat" > gpurun_out/r02t_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02t_tests.log
for sm in 1 0; do LG_SWEEP_SMALL=$sm timeout 300 python scripts/ic0_time.py C1 C2 > gpurun_out/r02t_ic0_s$sm.txt 2>&1; echo "small=$sm: $(cat gpurun_out/r02t_ic0_s$sm.txt | tr '\n' ' ')"; done
for sm in 1 0; do LG_SWEEP_SMALL=$sm timeout 600 python scripts/small_solves.py > gpurun_out/r02t_solves_s$sm.jsonl 2>&1; echo "small=$sm:"; cat gpurun_out/r02t_solves_s$sm.jsonl; done
