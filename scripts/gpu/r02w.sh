timeout 600 python scripts/iter_roofline.py C4 --k 6 > gpurun_out/r02w_c4_ic0.json 2> gpurun_out/r02w_err.log; echo "rc=$?"; tail -3 gpurun_out/r02w_err.log
timeout 600 python scripts/iter_roofline.py C4 --k 6 --fsai > gpurun_out/r02w_c4_fsai.json 2>> gpurun_out/r02w_err.log; echo "rc=$?"
