#!/usr/bin/env bash
# Functional check of bench.py's N>1 path on a one-GPU box: two ranks share
# GPU 0 over a gloo group (timing is not meaningful, the plumbing is).
O=gpurun_out/${1:-r2}; mkdir -p $O
PORT=29533
for r in 0 1; do
  WORLD_SIZE=2 RANK=$r LOCAL_RANK=0 MASTER_ADDR=127.0.0.1 MASTER_PORT=$PORT PRRTC_BENCH_BACKEND=gloo \
    timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --latency-samples 10 \
    > $O/rank$r.json 2> $O/rank$r.err &
done
wait
