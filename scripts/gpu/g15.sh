# round-2 call (4 GPUs): op windows (64 KiB / 256 KiB per CTA) at the 1 GiB headline and at N=1
mkdir -p gpurun_out
run() { timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare "${@:2}" 2>> gpurun_out/g15.err | tail -1; }
for mcb in 0 65536 262144; do
  echo "{\"n\":1,\"mcb\":$mcb,\"line\":$(THEMIS_MIN_CTA_BYTES=$mcb timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare 2>>gpurun_out/g15.err | tail -1)}" >> gpurun_out/g15.jsonl
  echo "{\"n\":1,\"mcb\":$mcb,\"ratio\":\"1:1:1\",\"line\":$(THEMIS_MIN_CTA_BYTES=$mcb timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare --ratio 1:1:1 2>>gpurun_out/g15.err | tail -1)}" >> gpurun_out/g15.jsonl
  echo "{\"n\":4,\"mcb\":$mcb,\"line\":$(THEMIS_MIN_CTA_BYTES=$mcb run 4)}" >> gpurun_out/g15.jsonl
  echo "{\"n\":4,\"mcb\":$mcb,\"sizes\":\"2,2\",\"line\":$(THEMIS_MIN_CTA_BYTES=$mcb run 4 --sizes 2,2 --ratio 1:1)}" >> gpurun_out/g15.jsonl
  echo "{\"n\":2,\"mcb\":$mcb,\"line\":$(THEMIS_MIN_CTA_BYTES=$mcb run 2)}" >> gpurun_out/g15.jsonl
  echo "{\"n\":2,\"mcb\":$mcb,\"la\":1,\"line\":$(THEMIS_MIN_CTA_BYTES=$mcb run 2 --lookahead 1)}" >> gpurun_out/g15.jsonl
done
