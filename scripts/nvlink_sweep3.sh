#!/bin/bash
N=$1; OUT=$2; mkdir -p $OUT
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu "$@"; }
for ct in 32 64 148; do for ch in 8 64; do
  run --no-compare --sizes $N --ratio 1 --chunks $ch --ctas-total $ct > $OUT/flat_c${ct}_ch$ch.json 2>/dev/null
done; done
run --sizes 2,2 --ratio 2:1 --compare-ratios 1:1 --ctas-total 64 > $OUT/2x2_c64.json 2>/dev/null
run > $OUT/2x2x2_default.json 2>/dev/null
