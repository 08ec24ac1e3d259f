# alternate variant libraries R times on one config (noise control): gpu_alt.sh CONFIG R v1 v2 ...
mkdir -p gpurun_out
c=$1; R=$2; shift 2
for r in $(seq 1 $R); do for v in "$@"; do
  SUBSURF_B200_LIB=variants/$v.so timeout 120 python scripts/sweep_rate.py $c | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', $r, d['us_per_sweep'])" >> gpurun_out/alt_$c.txt 2>&1
done; done
