#!/bin/bash
N=$1; OUT=$2; mkdir -p $OUT
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu --no-compare "$@"; }
for st in 3 4 6; do for ct in 32 48 64 96; do
  run --sizes 2,2 --ratio 2:1 --stages $st --ctas-total $ct > $OUT/2x2_s${st}_c${ct}.json 2>/dev/null
  run --sizes 2,2 --ratio 1:1 --stages $st --ctas-total $ct > $OUT/2x2_11_s${st}_c${ct}.json 2>/dev/null
done; done
