# round-2 call (4 GPUs): NVLS dims with the runtime order -- parity (mp_worker NVLS cases) and flat / 2x4 throughput
mkdir -p gpurun_out
for n in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n tests/mp_worker.py > gpurun_out/g21_multi_w$n.log 2>&1; echo "rc=$?" >> gpurun_out/g21_multi_w$n.log; done
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare --nccl "$@" 2>> gpurun_out/g21.err | tail -1; }
for la in 1 16; do
  echo "{\"t\":\"flat_nvls\",\"la\":$la,\"line\":$(run --sizes 4 --ratio 1 --nvls --lookahead $la)}" >> gpurun_out/g21.jsonl
  echo "{\"t\":\"2x4_nvls\",\"la\":$la,\"line\":$(run --sizes 2,4 --ratio 1:1 --nvls --lookahead $la)}" >> gpurun_out/g21.jsonl
  echo "{\"t\":\"flat_nvls_c16\",\"la\":$la,\"line\":$(run --sizes 4 --ratio 1 --nvls --lookahead $la --chunks 16)}" >> gpurun_out/g21.jsonl
done
echo "{\"t\":\"2x4\",\"la\":16,\"line\":$(run --sizes 2,4 --ratio 1:1)}" >> gpurun_out/g21.jsonl
echo "{\"t\":\"flat\",\"la\":16,\"line\":$(run --sizes 4 --ratio 1 --chunks 16)}" >> gpurun_out/g21.jsonl
