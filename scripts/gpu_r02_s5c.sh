#!/bin/bash
# session 5: hunt the 3-rank bench hang (host transport): repeat the torchrun line with the watchdog on
mkdir -p gpurun_out
for i in 1 2 3 4 5 6 7 8 9 10; do
  t0=$(date +%s)
  SUBSURF_DIST_TRANSPORT=host SUBSURF_BENCH_WATCHDOG=120 timeout -k 5 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=3 \
    --master-addr 127.0.0.1 --master-port $((29500 + i)) bench.py --gpus 3 --config tiny --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/s5c_run$i.out 2> gpurun_out/s5c_run$i.err
  echo "run $i rc=$? $(( $(date +%s) - t0 )) s" | tee -a gpurun_out/s5c_summary.txt
done
nvidia-smi --query-compute-apps=pid,used_memory --format=csv | tee -a gpurun_out/s5c_summary.txt
