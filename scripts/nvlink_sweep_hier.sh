#!/bin/bash
# Hierarchical NVLink calibration: 2x2 logical topology, one rank per GPU (4 GPUs),
# busBW vs CTA budget x TMA ring depth x stage size.  Usage: scripts/nvlink_sweep_hier.sh OUTDIR
OUT=$1; mkdir -p $OUT
run() { timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu --no-compare --sizes 2,2 "$@"; }
for kb in 32 16; do for st in 2 3 4 6; do for ct in 48 64 96 128 148; do
  [ $kb -eq 16 ] && [ $st -lt 4 ] && continue
  run --ratio 2:1 --ctas-total $ct --stages $st --stage-kb $kb > $OUT/2x2_kb${kb}_s${st}_c${ct}.json 2>/dev/null
  echo "kb=$kb st=$st ct=$ct $(python3 -c "import json,sys; print(json.loads(open('$OUT/2x2_kb${kb}_s${st}_c${ct}.json').read().strip().splitlines()[-1])['value'])" 2>&1 | tail -1)"
done; done; done
