# round-2 call (4 GPUs): config-4 DDP buckets and config-3 with runtime order (auto L=16 at N=4) + latency-aware auto chunks
mkdir -p gpurun_out
run() { timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) "${@:2}"; }
run 4 scripts/sweeps.py --config 4 --quick --latency-ns 11000 > gpurun_out/g18_cfg4_n4.jsonl 2> gpurun_out/g18.err
run 4 scripts/sweeps.py --config 3 --quick --latency-ns 11000 > gpurun_out/g18_cfg3_n4.jsonl 2>> gpurun_out/g18.err
