# IC(0) dataflow sweep knobs: staggered polling, reciprocal multiply, gate
for v in default poll100 poll250 rcp; do
  if [ $v = default ]; then ov=""; else ov="build/variants/$v.so"; fi
  LG_LIB_OVERRIDE=$ov timeout 300 python scripts/flow_trace.py C4 > gpurun_out/r02p_$v.txt 2>&1
  echo "$v: $(grep -E 'fwd:|bwd:' gpurun_out/r02p_$v.txt | sed 's/tasks.*span/span/' | tr '\n' ' ')"
done
for g in 1 2 5; do
  LG_SWEEP_GATE=$g timeout 300 python scripts/flow_trace.py C4 > gpurun_out/r02p_g$g.txt 2>&1
  echo "gate $g: $(grep -E 'fwd:|bwd:' gpurun_out/r02p_g$g.txt | sed 's/tasks.*span/span/' | tr '\n' ' ')"
done
