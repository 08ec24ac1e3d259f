#!/bin/bash
# item order A/B on config 4 (power-capped loop) + ncu DRAM bytes of a red pass per order
mkdir -p gpurun_out
O=gpurun_out/order_m.jsonl
for r in 1 2; do
for o in 1 2; do
  SSB_ORDER=$o timeout 300 python scripts/power_probe.py config4 | sed "s/\"config\"/\"order\": $o, \"config\"/" >> $O 2>&1
done
done
SSB_ORDER=2 timeout 900 bash scripts/ncu_pass.sh config4 c4_red_order2
cat $O
