#!/bin/bash
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) "$@"; }
for rr in 0 1; do
  echo "== AG_RR=$rr"
  THEMIS_AG_RR=$rr run scripts/latency_probe.py --sizes 4 --ctas 32 --mib 1024 2>&1 | grep -E "dim1|kernel"
  THEMIS_AG_RR=$rr run bench.py --gpus 4 --sizes 4 --ratio 1 --no-e2e --no-cpu --no-compare 2>/dev/null | cut -c1-140
  THEMIS_AG_RR=$rr run bench.py --gpus 4 --sizes 2,2 --ratio 2:1 --no-e2e --no-cpu --no-compare 2>/dev/null | cut -c1-140
done
