#!/bin/bash
N=$1; OUT=$2; mkdir -p $OUT
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu --no-compare "$@"; }
for kb in 16 32 64; do for st in 2 3 4 6 8 12; do
  if [ $((kb * st)) -gt 192 ]; then continue; fi
  run --sizes 2,2 --ratio 2:1 --stages $st --stage-kb $kb --ctas-total 48 > $OUT/2x2_kb${kb}_s${st}.json 2>/dev/null
  run --sizes 4 --ratio 1 --stages $st --stage-kb $kb --ctas-total 32 > $OUT/flat_kb${kb}_s${st}.json 2>/dev/null
done; done
