#!/bin/bash
# ncu_pass.sh CONFIG OUT [kernel-regex] [skip] : one --set full capture of a red TMA pass of
# scripts/sweep_rate.py CONFIG -> gpurun_out/OUT.ncu-rep.  skip (default 5) matching launches
# first: the first pass of a solve reads its guess buffer twice (it IS the rhs), later
# passes are the steady state.
K=${3:-'regex:sor_pass_tma<\(int\)0, \(bool\)0, \(bool\)0, \(bool\)1>'}
SKIP=${4:-5}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" -s $SKIP -c 1 \
    -o gpurun_out/$2 -f python scripts/sweep_rate.py $1 > gpurun_out/$2.log 2>&1
