for v in default poll1; do
  if [ $v = default ]; then ov=""; else ov="build/variants/$v.so"; fi
  LG_LIB_OVERRIDE=$ov timeout 300 python scripts/flow_trace.py C4 C3 > gpurun_out/r02q_$v.txt 2>&1
  echo "$v: $(grep -E 'fwd:|bwd:' gpurun_out/r02q_$v.txt | sed 's/tasks.*span/span/' | tr '\n' ' ')"
done
LG_SWEEP_BACKOFF=64 timeout 300 python scripts/flow_trace.py C4 > gpurun_out/r02q_bo64.txt 2>&1
echo "backoff64: $(grep -E 'fwd:|bwd:' gpurun_out/r02q_bo64.txt | sed 's/tasks.*span/span/' | tr '\n' ' ')"
