#!/bin/bash
# All-NVLink hierarchical (2x2, one rank per GPU, 4 GPUs): CTA budget x ring shape, 3 repeats.
val() { python3 -c "import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])['value'])" 2>&1 | tail -1; }
for cfg in "96 3 32" "128 2 32" "96 2 48" "128 2 48" "64 3 64" "96 2 64" "128 3 32"; do set -- $cfg
  r=""
  for rep in 1 2 3; do
    r="$r $(timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --sizes 2,2 --ratio 2:1 --no-e2e --no-cpu --no-compare --ctas-total $1 --stages $2 --stage-kb $3 2>/dev/null | val)"
  done
  echo "ctas $1 stages $2 x $3 KiB:$r"
done
