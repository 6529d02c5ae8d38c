# chunked exact degrees, panelled exterior halves: tests, C5 projection, build launch list
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > gpurun_out/r02ad_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02ad_tests.log
timeout 1500 python scripts/scaling_projection.py C5 --jacobi --device-collectives > gpurun_out/r02ad_proj_c5.jsonl 2>&1; echo "proj c5 rc=$?"
python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02ad_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ad_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02ad_ncu1.log 2>&1; echo "launches rc=$?"
