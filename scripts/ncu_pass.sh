#!/bin/bash
# ncu_pass.sh CONFIG OUT [kernel-regex] : one --set full capture of the first red TMA pass
# (after prepare) of scripts/sweep_rate.py CONFIG -> gpurun_out/OUT.ncu-rep
K=${3:-'regex:sor_pass_tma<\(int\)0, \(bool\)0>'}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -c 1 \
    -o gpurun_out/$2 -f python scripts/sweep_rate.py $1 > gpurun_out/$2.log 2>&1
