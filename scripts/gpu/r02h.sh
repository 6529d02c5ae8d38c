python scripts/spmv_ab.py C4 > gpurun_out/r02h_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wspmv -s 5 -c 1 \
  -o gpurun_out/r02h_wspmv python scripts/spmv_ab.py C4 > gpurun_out/r02h_ncu.log 2>&1
echo "rc=$?"
