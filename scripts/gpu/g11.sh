# round-2 call (4 GPUs): small-collective regime (A_K): static vs runtime order, fixed 64 vs planner-chosen chunks, NCCL beside
mkdir -p gpurun_out
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu --no-compare --nccl "$@" 2>> gpurun_out/g11.err | tail -1; }
for mib in 1 4 16 64 256; do
  for sz in "2,2,2 4:2:1" "2,2 1:1"; do set -- $sz
    for la in 1 16; do
      for ch in 64 8; do
        echo "{\"mib\":$mib,\"sizes\":\"$1\",\"la\":$la,\"chunks\":$ch,\"line\":$(run --sizes $1 --ratio $2 --mib $mib --chunks $ch --lookahead $la)}" >> gpurun_out/g11.jsonl
      done
    done
  done
done
