#!/bin/bash
# K5-style calibration: NVLink-only (one logical rank per GPU) All-Reduce busBW
# vs CTAs per dimension group.  Usage: scripts/nvlink_sweep.sh N OUTDIR
N=$1; OUT=$2; mkdir -p $OUT
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu "$@"; }
for ct in 8 16 32 64 148; do
  run --sizes $N --ratio 1 --ctas-total $ct --no-compare > $OUT/flat_n${N}_c${ct}.json 2>/dev/null
done
if [ $N -eq 4 ]; then
  run --sizes 2,2 --ratio 2:1 --compare-ratios 1:1 > $OUT/2x2_n4.json 2>/dev/null
  run --sizes 2,2 --ratio 2:1 --compare-ratios 1:1 --ctas-total 32 > $OUT/2x2_n4_c32.json 2>/dev/null
fi
