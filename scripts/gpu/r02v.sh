# per-launch duration + DRAM bytes of one C4 DACG iteration (reference IC(0)), and of one
# FSAI iteration; event-timed iteration for the per-iteration GB/s
python scripts/prof_iter.py C4 --k 6 > gpurun_out/r02v_plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/r02v_iter_c4.csv python scripts/prof_iter.py C4 --k 6 > gpurun_out/r02v_ncu.log 2>&1; echo "ncu rc=$?"
timeout 300 python scripts/dacg_iter.py C4 > gpurun_out/r02v_dacg_iter.txt 2>&1; echo "iter rc=$?"; tail -5 gpurun_out/r02v_dacg_iter.txt
