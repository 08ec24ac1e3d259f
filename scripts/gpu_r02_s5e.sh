#!/bin/bash
# session 5: stress the 3-rank bench line (host transport) to catch the rare hang: 45 runs, watchdog 60 s
mkdir -p gpurun_out
for i in $(seq 1 45); do
  t0=$(date +%s)
  SUBSURF_DIST_TRANSPORT=host SUBSURF_BENCH_WATCHDOG=60 timeout -k 5 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node=3 \
    --master-addr 127.0.0.1 --master-port $((29600 + i)) bench.py --gpus 3 --config tiny --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/s5e_run.out 2> gpurun_out/s5e_run.err
  rc=$?
  echo "run $i rc=$rc $(( $(date +%s) - t0 )) s" >> gpurun_out/s5e_summary.txt
  if [ $rc -ne 0 ]; then cp gpurun_out/s5e_run.err gpurun_out/s5e_fail$i.err; cp gpurun_out/s5e_run.out gpurun_out/s5e_fail$i.out; fi
done
grep -c "rc=0" gpurun_out/s5e_summary.txt; grep -v "rc=0" gpurun_out/s5e_summary.txt
