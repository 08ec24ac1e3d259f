#!/bin/bash
# certified face gradients: parity tests, assembly ms per step with / without, bench config 4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "certified or tile_assembly or assemble" > gpurun_out/cert_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cert_tests.log
grep -E "no-margin|passed|failed|rc=" gpurun_out/cert_tests.log
O=gpurun_out/asm_cert.jsonl
for c in config1 config4; do
  for v in 1 0 1 0; do
    SSB_ASM_CERT=$v timeout 300 python scripts/asm_rate.py $c | sed "s/\"config\"/\"cert\": $v, \"config\"/" >> $O 2>&1
  done
done
cut -c1-160 $O
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_c4_za.json 2> gpurun_out/bench_c4_za.err
python -c "import json; d=json.load(open('gpurun_out/bench_c4_za.json')); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('assemble_ms_per_step'), d['clocks'])"
