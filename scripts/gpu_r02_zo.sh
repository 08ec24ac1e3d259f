#!/bin/bash
mkdir -p gpurun_out
for v in nb4g3pad nb4g2pad; do
  echo "== $v"; SUBSURF_B200_LIB=variants/$v.so timeout 120 python scripts/asm_rate.py config0 2>&1 | tail -1 | cut -c1-150
done
python - <<'PY'
import torch, ctypes
print(torch.cuda.get_device_properties(0))
PY
