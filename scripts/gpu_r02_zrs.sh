#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python scripts/rank_share_rate.py 8 4 2 > gpurun_out/rank_share.jsonl 2> gpurun_out/rank_share.err
cat gpurun_out/rank_share.jsonl; tail -3 gpurun_out/rank_share.err
