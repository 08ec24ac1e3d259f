#!/bin/bash
mkdir -p gpurun_out
timeout 300 python scripts/sustained_copy.py > gpurun_out/sustained_copy.json 2>&1; cat gpurun_out/sustained_copy.json
timeout 300 python scripts/power_probe.py config4 > gpurun_out/power_c4_r.json 2>&1; cat gpurun_out/power_c4_r.json
timeout 300 python scripts/sustained_copy.py >> gpurun_out/sustained_copy.json 2>&1; tail -1 gpurun_out/sustained_copy.json
