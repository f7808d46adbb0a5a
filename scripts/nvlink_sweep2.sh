#!/bin/bash
N=$1; OUT=$2; mkdir -p $OUT
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu --no-compare --sizes $N --ratio 1 "$@"; }
for ch in 8 64; do
  run --chunks $ch --ctas-total 64 > $OUT/tma_c64_ch$ch.json 2>/dev/null
  THEMIS_COPY_ENGINE=ldg run --chunks $ch --ctas-total 64 > $OUT/ldg_c64_ch$ch.json 2>/dev/null
  THEMIS_COPY_ENGINE=ldg run --chunks $ch --ctas-total 148 > $OUT/ldg_c148_ch$ch.json 2>/dev/null
done
run --chunks 64 --ctas-total 64 --mib 4096 > $OUT/tma_c64_4g.json 2>/dev/null
