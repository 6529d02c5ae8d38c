# medium-row blocks: correctness + A/B vs no-med (p1m4), then ncu of med on C4
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "spmv or row_part or laplacian or spmm" > gpurun_out/r02n_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02n_tests.log
for v in med p1m4; do
  LG_LIB_OVERRIDE=build/variants/$v.so timeout 300 python scripts/spmv_ab.py C3 C4 C5 > gpurun_out/r02n_$v.jsonl 2>&1; echo "$v: $(python -c "
import json
for l in open('gpurun_out/r02n_$v.jsonl'):
    try: d=json.loads(l); print(d['graph'], round(d['us'],1), end='  ')
    except Exception: pass
")"
done
python scripts/spmv_ab.py C4 > gpurun_out/r02n_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:wspmv -s 5 -c 1 \
  -o gpurun_out/r02n_wspmv python scripts/spmv_ab.py C4 > gpurun_out/r02n_ncu.log 2>&1
echo "ncu rc=$?"
