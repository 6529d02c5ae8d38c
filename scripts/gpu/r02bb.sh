# R-MAT ladder with the level-merged sweeps (scale 20 and 22, with solves), and the plain sweeps for the apply time
timeout 900 python scripts/ic0_ladder.py 20 --solve > gpurun_out/r02g_ic0_ladder_s20.jsonl 2>&1; tail -1 gpurun_out/r02g_ic0_ladder_s20.jsonl | cut -c1-900
LG_IC0_MERGE=0 timeout 900 python scripts/ic0_ladder.py 20 > gpurun_out/r02g_ic0_ladder_s20_plain.jsonl 2>&1; tail -1 gpurun_out/r02g_ic0_ladder_s20_plain.jsonl | cut -c1-600
timeout 1500 python scripts/ic0_ladder.py 22 --solve > gpurun_out/r02g_ic0_ladder_s22.jsonl 2>&1; tail -1 gpurun_out/r02g_ic0_ladder_s22.jsonl | cut -c1-900
# refreshed full capture of the merged sweep (hub ordering, wide CTA)
python scripts/ic0_time.py C4 > gpurun_out/r02g_ic0_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_flow -s 6 -c 2 -o gpurun_out/r02g_sweep \
  python scripts/ic0_time.py C4 > gpurun_out/r02g_ncu3.log 2>&1; echo "ncu sweep rc=$?"
ncu --page details --csv -i gpurun_out/r02g_sweep.ncu-rep > gpurun_out/r02g_sweep_details.csv 2>/dev/null
