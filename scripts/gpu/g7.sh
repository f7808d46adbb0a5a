# round-2 call (4 GPUs): bisect the static-order NVLink regression with THEMIS_EXP bits
mkdir -p gpurun_out
R=$PWD
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare "$@" 2>/dev/null | tail -1; }
for sz in "2,2 1:1" "2,4 1:1"; do set -- $sz
  echo "{\"tag\":\"old\",\"sizes\":\"$1\",\"line\":$(cd $R/old_227d847 && run --sizes $1 --ratio $2)}" >> gpurun_out/g7.jsonl
  for e in 0 1 2 4 8 15; do
    echo "{\"tag\":\"exp$e\",\"sizes\":\"$1\",\"line\":$(THEMIS_EXP=$e run --sizes $1 --ratio $2)}" >> gpurun_out/g7.jsonl
  done
done
