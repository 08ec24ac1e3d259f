#!/bin/bash
# 5 main-ring stages vs 4 under the power cap, configs 4 / 2 / 1, three alternating runs
mkdir -p gpurun_out
O=gpurun_out/power_ms5.jsonl; rm -f $O
for c in config4 config2 config1; do
  for rep in 1 2 3; do for v in base ms5; do
    if [ $v = base ]; then L=; else L=variants/$v.so; fi
    SUBSURF_B200_LIB=$L timeout 300 python scripts/power_probe.py $c 2>&1 | tail -1 | sed "s/\"config\"/\"var\": \"$v\", \"config\"/" >> $O
  done; done
done
python - <<'PY'
import json, collections
d=collections.defaultdict(list)
for l in open('gpurun_out/power_ms5.jsonl'):
    if l.startswith('{'):
        r=json.loads(l); d[(r['config'], r['var'])].append(r['us_per_sweep'])
for k,v in sorted(d.items()): print(k, [round(x,1) for x in v])
PY
