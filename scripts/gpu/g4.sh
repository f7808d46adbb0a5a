# round-2 call (4 GPUs): full GPU suite incl. multi-GPU; runtime intra-dim order on NVLink topologies
mkdir -p gpurun_out
python scripts/nvml_nvlink.py > gpurun_out/g4_nvml.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g4_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g4_pytest.log
run() { timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu "$@"; }
for la in 1 4 16; do
  run --sizes 2,2 --ratio 1:1 --lookahead $la >> gpurun_out/g4_bench.jsonl 2>> gpurun_out/g4_bench.err
  run --sizes 2,4 --ratio 1:1 --lookahead $la >> gpurun_out/g4_bench.jsonl 2>> gpurun_out/g4_bench.err
  run --lookahead $la --ratio 1:1:1 >> gpurun_out/g4_bench.jsonl 2>> gpurun_out/g4_bench.err
done
python scripts/nvml_nvlink.py >> gpurun_out/g4_nvml.txt 2>&1
