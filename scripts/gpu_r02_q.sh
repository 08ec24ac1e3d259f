#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/kw_q.jsonl
timeout 300 python scripts/sweep_rate.py config4 >> $O 2>&1
for v in kwp16l3 kwp16l3h3 kwp16l3h5 kwp16l3h7 kwp16l5h7 kwp32l3h1; do
  SUBSURF_B200_LIB=variants/$v.so SUBSURF_KERNEL=kwave timeout 300 python scripts/sweep_rate.py config4 | sed "s/\"config\"/\"variant\": \"$v\", \"config\"/" >> $O 2>&1
done
cut -c1-200 $O
