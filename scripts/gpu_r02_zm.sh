#!/bin/bash
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python scripts/asm_rate.py config0 > gpurun_out/san_col.log 2>&1
grep -v "^=========     \(Host\|#\)" gpurun_out/san_col.log | head -40
