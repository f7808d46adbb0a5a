#!/bin/bash
N=$1; OUT=$2; mkdir -p $OUT
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu "$@"; }
for st in 2 4 6; do for ct in 16 24 32 48; do
  THEMIS_STAGES=$st run --no-compare --sizes $N --ratio 1 --chunks 64 --ctas-total $ct > $OUT/flat_s${st}_c${ct}.json 2>/dev/null
done; done
for ct in 24 32 48 64 96; do
  run --no-compare --ctas-total $ct > $OUT/2x2x2_c${ct}.json 2>/dev/null
done
