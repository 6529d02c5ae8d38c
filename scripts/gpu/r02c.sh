# ncu --set full of the warp-block SpMV on C4
python scripts/spmv_ab.py C4 > gpurun_out/r02c_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wspmv -s 5 -c 1 \
  -o gpurun_out/r02c_wspmv python scripts/spmv_ab.py C4 > gpurun_out/r02c_ncu.log 2>&1
echo "rc=$?"
