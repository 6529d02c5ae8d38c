python scripts/gpu/nsres.py 2>&1 | tail -5
timeout 300 python scripts/dacg_iter.py C1 > gpurun_out/r02ac_c1.txt 2>&1; cat gpurun_out/r02ac_c1.txt
timeout 300 python scripts/dacg_iter.py C2 > gpurun_out/r02ac_c2.txt 2>&1; cat gpurun_out/r02ac_c2.txt
