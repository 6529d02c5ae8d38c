# resident one-CTA IC(0) sweep, cp.async-staged: parity tests and timing
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "ic0" > gpurun_out/r02aj_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r02aj_tests.log
rm -f gpurun_out/r02aj_modes.jsonl
for th in 512 768 256; do
  LG_SWEEP_CTA_THREADS=$th timeout 300 python scripts/ic0_modes.py C1 C2 C3 >> gpurun_out/r02aj_modes.jsonl 2>&1
done
cat gpurun_out/r02aj_modes.jsonl
LG_SWEEP_CTA=1 timeout 300 python scripts/flow_trace.py C1 C2 > gpurun_out/r02aj_trace.txt 2>&1; cat gpurun_out/r02aj_trace.txt
