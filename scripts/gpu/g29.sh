# round-2 call (4 GPUs): A/B of the default N=4 / N=1 bench, HEAD vs f6b4632 (before push-pipelining / NVLS runtime order / LL)
mkdir -p gpurun_out
R=$PWD
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-compare --no-e2e --no-cpu 2>/dev/null | tail -1; }
for rep in 1 2; do
  echo "{\"tag\":\"head_n4\",\"line\":$(run)}" >> gpurun_out/g29.jsonl
  echo "{\"tag\":\"old_n4\",\"line\":$(cd $R/old_f6b && run)}" >> gpurun_out/g29.jsonl
  echo "{\"tag\":\"head_n1\",\"line\":$(timeout 300 python bench.py --steps 10 --warmup 3 --no-compare --no-e2e --no-cpu 2>/dev/null | tail -1)}" >> gpurun_out/g29.jsonl
  echo "{\"tag\":\"old_n1\",\"line\":$(cd $R/old_f6b && timeout 300 python bench.py --steps 10 --warmup 3 --no-compare --no-e2e --no-cpu 2>/dev/null | tail -1)}" >> gpurun_out/g29.jsonl
done
