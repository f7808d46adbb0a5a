# round-2 call (4 GPUs): warp-parallel readiness scan -- N=2/4 headline, small collectives with windows
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "runtime or random_executor or push" > gpurun_out/g16_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g16_pytest.log
run() { timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare "${@:2}" 2>> gpurun_out/g16.err | tail -1; }
for rep in 1 2; do
for la in 1 16; do
  echo "{\"n\":2,\"la\":$la,\"line\":$(run 2 --lookahead $la)}" >> gpurun_out/g16.jsonl
  echo "{\"n\":4,\"la\":$la,\"line\":$(run 4 --lookahead $la)}" >> gpurun_out/g16.jsonl
  echo "{\"n\":4,\"la\":$la,\"sizes\":\"2,2\",\"line\":$(run 4 --lookahead $la --sizes 2,2 --ratio 1:1)}" >> gpurun_out/g16.jsonl
done; done
for la in 1 16; do for sz in "2,2,2 4:2:1" "2,2 1:1"; do set -- $sz
  echo "{\"n\":4,\"la\":$la,\"mib\":16,\"sizes\":\"$1\",\"line\":$(THEMIS_MIN_CTA_BYTES=65536 run 4 --lookahead $la --sizes $1 --ratio $2 --mib 16 --chunks 64)}" >> gpurun_out/g16.jsonl
done; done
