# resident one-CTA IC(0) sweep: parity tests and timing against the dataflow sweeps
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "ic0" > gpurun_out/r02ag_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/r02ag_tests.log
for th in 512 256 128; do
  LG_SWEEP_CTA_THREADS=$th timeout 300 python scripts/ic0_modes.py C1 C2 C3 >> gpurun_out/r02ag_modes.jsonl 2>&1
done
cat gpurun_out/r02ag_modes.jsonl
