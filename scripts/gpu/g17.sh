# round-2 call (4 GPUs): bench lines with the round-2 defaults at N=1/2/4; config-3/4 sweeps at N=4 (NCCL rows beside)
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g17_n1.json 2> gpurun_out/g17.err
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) "${@:2}"; }
run 4 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/g17_n4.json 2>> gpurun_out/g17.err
run 2 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/g17_n2.json 2>> gpurun_out/g17.err
run 4 bench.py --gpus 4 --steps 20 --warmup 5 --sizes 2,2 --ratio 1:1 --no-e2e --pace-gbs 600 > gpurun_out/g17_n4_2x2.json 2>> gpurun_out/g17.err
run 4 scripts/sweeps.py --config 3 --quick > gpurun_out/g17_cfg3_n4.jsonl 2>> gpurun_out/g17.err
run 4 scripts/sweeps.py --config 4 --quick > gpurun_out/g17_cfg4_n4.jsonl 2>> gpurun_out/g17.err
