#!/bin/bash
mkdir -p gpurun_out
SUBSURF_B200_LIB=variants/kwp16l3.so SUBSURF_KERNEL=kwave timeout 900 bash scripts/ncu_pass.sh config4 kwp16_c4 'regex:sor_kwave_tma' 3
ls -la gpurun_out/kwp16_c4.ncu-rep
