#!/bin/bash
# parameter sweep of the SOR pass under the power cap (config 4): L2 policies, ring depths, item hand-out
mkdir -p gpurun_out
O=gpurun_out/power_sweep.jsonl; rm -f $O
run() { SUBSURF_B200_LIB=$2 timeout 300 env $3 python scripts/power_probe.py config4 2>&1 | tail -1 | sed "s/\"config\"/\"var\": \"$1\", \"config\"/" >> $O; }
for rep in 1 2; do
  run base "" "X=0"
  run l2h1 "" "SSB_L2HINT=1"
  run l2h3 "" "SSB_L2HINT=3"
  run l2h5 "" "SSB_L2HINT=5"
  for v in ms3 ms5 uk5 uk8 nodyn; do run $v variants/$v.so "X=0"; done
done
cut -c1-170 $O
