#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/kw_o.jsonl
timeout 300 python scripts/sweep_rate.py config4 >> $O 2>&1
for v in kwp8l2 kwp8l3 kwp16l2 kwp16l3; do
  SUBSURF_B200_LIB=variants/$v.so SUBSURF_KERNEL=kwave timeout 300 python scripts/sweep_rate.py config4 | sed "s/\"config\"/\"variant\": \"$v\", \"config\"/" >> $O 2>&1
done
CHECK_VS_TMA=1 SUBSURF_B200_LIB=variants/kwp16l2.so SUBSURF_KERNEL=kwave timeout 300 python scripts/sweep_rate.py config4 >> $O 2>&1
cat $O
