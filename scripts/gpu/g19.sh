# round-2 call (4 GPUs): CTA split for throughput at N=2 / N=4 (headline plan), stages
mkdir -p gpurun_out
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare "${@:2}" 2>> gpurun_out/g19.err | tail -1; }
for sp in 85,42,21 74,37,37 66,33,49 60,44,44 50,49,49; do
  echo "{\"n\":2,\"split\":\"$sp\",\"line\":$(run 2 --ctas-split $sp)}" >> gpurun_out/g19.jsonl
done
for sp in 55,27,14 48,24,24 40,28,28 32,32,32 64,42,42; do
  echo "{\"n\":4,\"split\":\"$sp\",\"line\":$(run 4 --ctas-split $sp)}" >> gpurun_out/g19.jsonl
done
for st in "3 64" "6 32" "2 96"; do set -- $st
  echo "{\"n\":2,\"stages\":\"$1x$2\",\"line\":$(run 2 --stages $1 --stage-kb $2)}" >> gpurun_out/g19.jsonl
done
