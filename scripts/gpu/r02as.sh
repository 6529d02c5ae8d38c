# round-2 final evidence (level-merged IC(0) sweeps, live gather floor): bench lines, reference arm,
# ncu launch list of the bench command, full ncu captures of the SpMV and the dataflow sweep, per-pass roofline
set -x
timeout 1500 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?"; head -c 600 gpurun_out/r02d_bench.json
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/r02d_bench_c5.json 2> gpurun_out/r02d_bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r02d_reference.json 2>&1; echo "reference rc=$?"
python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02d_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02d_ncu1.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:wspmv -s 3 -c 1 -o gpurun_out/r02d_spmv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02d_ncu2.log 2>&1; echo "ncu spmv rc=$?"
ncu --page details --csv -i gpurun_out/r02d_spmv.ncu-rep > gpurun_out/r02d_spmv_details.csv 2>/dev/null
python scripts/ic0_time.py C4 > gpurun_out/r02d_ic0_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_flow -s 6 -c 2 -o gpurun_out/r02d_sweep \
  python scripts/ic0_time.py C4 > gpurun_out/r02d_ncu3.log 2>&1; echo "ncu sweep rc=$?"
ncu --page details --csv -i gpurun_out/r02d_sweep.ncu-rep > gpurun_out/r02d_sweep_details.csv 2>/dev/null
timeout 600 python scripts/iter_roofline.py C4 > gpurun_out/r02d_iter_roofline_ic0.json 2> gpurun_out/r02d_iter_roofline_ic0.err; echo "iter roofline rc=$?"
timeout 300 python scripts/dacg_iter.py C4 > gpurun_out/r02d_dacg_iter_c4.txt 2>&1; cat gpurun_out/r02d_dacg_iter_c4.txt
timeout 300 python scripts/dacg_iter.py C1 > gpurun_out/r02d_dacg_iter_c1.txt 2>&1; cat gpurun_out/r02d_dacg_iter_c1.txt
timeout 300 python scripts/ic0_time.py C1 C2 C3 C4 > gpurun_out/r02d_ic0_time.txt 2>&1; cat gpurun_out/r02d_ic0_time.txt
rm -f gpurun_out/r02d_spmv.ncu-rep.tmp
ls -la gpurun_out/*.ncu-rep
