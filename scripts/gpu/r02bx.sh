# final bench lines with the NVML clock sampler
timeout 1500 python bench.py > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 > gpurun_out/r02m_bench_c5.json 2> gpurun_out/r02m_bench_c5.err; echo "bench c5 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r02m_reference.json 2>&1; echo "reference rc=$?"
