# slot-array finishing: A/B of occupancy / prefetch
for v in slot_m4 slot_m3; do
  LG_LIB_OVERRIDE=build/variants/$v.so timeout 300 python scripts/spmv_ab.py C3 C4 > gpurun_out/r02g_ab_$v.jsonl 2>&1; echo "$v rc=$?"; cat gpurun_out/r02g_ab_$v.jsonl
done
LG_SPMV_PREFETCH=0 LG_LIB_OVERRIDE=build/variants/slot_m4.so timeout 300 python scripts/spmv_ab.py C4 > gpurun_out/r02g_ab_nopf.jsonl 2>&1; echo "nopf rc=$?"; cat gpurun_out/r02g_ab_nopf.jsonl
