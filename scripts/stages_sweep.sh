#!/bin/bash
# TMA ring depth at N = 2 / 4 (mixed GPU-local + NVLink dims), headline config.
OUT=$1; mkdir -p $OUT
for n in 2 4; do for st in 3 4 6; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare --stages $st > $OUT/n${n}_s${st}.json 2>/dev/null
  echo "n=$n stages=$st $(python3 -c "import json; print(json.loads(open('$OUT/n${n}_s${st}.json').read().strip().splitlines()[-1])['value'])" 2>&1 | tail -1)"
done; done
