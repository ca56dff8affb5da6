#!/bin/bash
# per-rank work of an N-way vocabulary shard on one GPU (the NCCL exchanges excluded): V/N rows
for rows in 256000 128000 64000 32000; do
  timeout 300 python bench.py --no-cpu-baseline --vocab $rows --steps 20 --warmup 5 > gpurun_out/shard_$rows.json 2>/dev/null; echo rows=$rows rc=$?
done
