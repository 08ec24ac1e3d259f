mkdir -p gpurun_out
[ -n "$TESTS" ] && timeout 300 python -m pytest tests/test_gpu_slabs.py -x -q -k "kwave" > gpurun_out/kw_tests.log 2>&1
for v in "$@"; do
  SUBSURF_KERNEL=kwave SUBSURF_B200_LIB=variants/$v.so timeout 120 python scripts/sweep_rate.py config1 > gpurun_out/kwv_$v.json 2> gpurun_out/kwv_$v.err
done
