# round-2 call (4 GPUs): executor ceilings without dependencies (solo / all GPUs at once), paced budgets, latency breakdown
mkdir -p gpurun_out
K="timeout 180 python scripts/k5_nvlink.py --sizes 2,2 --mib 1024 --bw-gbs 1,1"
for la in 1 16; do for ct in "64,64" "74,74" "48,48"; do
  $K --ctas $ct --lookahead $la --tag solo_la${la}_c${ct} >> gpurun_out/g9_k5.jsonl 2>> gpurun_out/g9.err
  $K --ctas $ct --lookahead $la --all-gpus --tag all_la${la}_c${ct} >> gpurun_out/g9_k5.jsonl 2>> gpurun_out/g9.err
done; done
for st in "2 32" "3 32" "4 32" "2 48" "3 48"; do set -- $st
  $K --ctas 64,64 --lookahead 16 --all-gpus --stages $1 --stage-kb $2 --tag all_la16_s$1_kb$2 >> gpurun_out/g9_k5.jsonl 2>> gpurun_out/g9.err
done
run() { timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) "$@"; }
for pg in 480 600 720; do
  run bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu --sizes 2,2 --ratio 1:1 --lookahead 16 --pace-gbs $pg >> gpurun_out/g9_bench.jsonl 2>> gpurun_out/g9.err
done
for kib in 1024 16384; do
  run scripts/latency_probe.py --sizes 2,2 --kib $kib --chunks 64 --ctas 64,64 > gpurun_out/g9_lat_$kib.log 2>> gpurun_out/g9.err
done
