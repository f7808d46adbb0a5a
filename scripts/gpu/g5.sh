# round-2 call (4 GPUs): A/B of the NVLink-path regression (old 227d847 tree vs HEAD, slot-release variants)
mkdir -p gpurun_out
R=$PWD
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare "$@" 2>/dev/null | tail -1; }
for rep in 1 2; do
for sz in "2,2 1:1" "2,4 1:1"; do set -- $sz
  echo "{\"tag\":\"old\",\"sizes\":\"$1\",\"line\":$(cd $R/old_227d847 && run --sizes $1 --ratio $2)}" >> gpurun_out/g5.jsonl
  echo "{\"tag\":\"new_exp0\",\"sizes\":\"$1\",\"line\":$(THEMIS_EXP=0 run --sizes $1 --ratio $2)}" >> gpurun_out/g5.jsonl
  echo "{\"tag\":\"new_exp1\",\"sizes\":\"$1\",\"line\":$(THEMIS_EXP=1 run --sizes $1 --ratio $2)}" >> gpurun_out/g5.jsonl
  echo "{\"tag\":\"new_exp1_la16\",\"sizes\":\"$1\",\"line\":$(THEMIS_EXP=1 run --sizes $1 --ratio $2 --lookahead 16)}" >> gpurun_out/g5.jsonl
  echo "{\"tag\":\"old_base\",\"sizes\":\"$1\",\"line\":$(cd $R/old_227d847 && run --sizes $1 --ratio 2:1)}" >> gpurun_out/g5.jsonl
  echo "{\"tag\":\"new_exp1_base\",\"sizes\":\"$1\",\"line\":$(THEMIS_EXP=1 run --sizes $1 --ratio 2:1)}" >> gpurun_out/g5.jsonl
done; done
