# round-2 call (4 GPUs): small collectives -- op windows (min CTA bytes) with the runtime order
mkdir -p gpurun_out
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu --no-compare "$@" 2>> gpurun_out/g13.err | tail -1; }
for mib in 4 16 64; do
  for sz in "2,2,2 4:2:1" "2,2 1:1"; do set -- $sz
    for mcb in 0 16384 65536 262144; do
      for ch in 64 16; do
        echo "{\"mib\":$mib,\"sizes\":\"$1\",\"mcb\":$mcb,\"chunks\":$ch,\"line\":$(THEMIS_MIN_CTA_BYTES=$mcb run --sizes $1 --ratio $2 --mib $mib --chunks $ch)}" >> gpurun_out/g13.jsonl
      done
    done
  done
done
