#!/bin/bash
# NVLink transfer-engine sweep (run under gpurun --gpus 4); one JSON line per point.
set -u
cd "$(dirname "$0")"
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o nvlink_probe nvlink_probe.cu || exit 1
OUT=${1:-/dev/stdout}
run() { timeout 60 ./nvlink_probe "$@" >> "$OUT" 2>&1 || echo "{\"failed\":\"$*\"}" >> "$OUT"; }
for pat in pair1 pair2 all; do run memcpy $pat 1 1 32 512 5; done
run local self 148 4 32 1024 5
for mode in pull push; do
  for pat in pair1 all mix; do
    for ctas in 16 32 64 128; do
      for shape in "2 32" "4 32" "3 64" "6 32"; do
        run $mode $pat $ctas $shape 512 5
      done
    done
  done
done
for ctas in 32 64 128; do run pushst all $ctas 4 32 512 5; done
