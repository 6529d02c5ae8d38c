timeout 600 python bench.py --no-solve --no-cpu --no-c5 --no-vendor > gpurun_out/r02bv_bench.json 2> gpurun_out/r02bv_bench.err; echo "rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/r02bv_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['clocks'])"; tail -3 gpurun_out/r02bv_bench.err
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu > gpurun_out/r02bv_bench_c5.json 2> gpurun_out/r02bv_bench_c5.err; python -c "
import json; d=json.loads(open('gpurun_out/r02bv_bench_c5.json').read().strip().splitlines()[-1]); print(d['value'], d['clocks'])"
