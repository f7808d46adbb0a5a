# round-2 call (4 GPUs): GPU suite + bench lines after the single-lane fence fix (static vs runtime order)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g8_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g8_pytest.log
run() { timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu "$@"; }
for la in 1 16; do
  run --sizes 2,2 --ratio 1:1 --lookahead $la >> gpurun_out/g8_bench.jsonl 2>> gpurun_out/g8_bench.err
  run --sizes 2,4 --ratio 1:1 --lookahead $la >> gpurun_out/g8_bench.jsonl 2>> gpurun_out/g8_bench.err
  run --lookahead $la --ratio 1:1:1 >> gpurun_out/g8_bench.jsonl 2>> gpurun_out/g8_bench.err
  timeout 400 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --lookahead $la >> gpurun_out/g8_bench_n1.jsonl 2>> gpurun_out/g8_bench.err
done
