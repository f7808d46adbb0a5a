set -x
nvidia-smi topo -m > gpurun_out/g1_topo.txt 2>&1
bash scripts/nvlink/sweep.sh $PWD/gpurun_out/g1_probe.jsonl > gpurun_out/g1_sweep.log 2>&1
for sz in "2,2 1:1" "4,2 1:1" "2,4 1:1"; do set -- $sz
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 --sizes $1 --ratio $2 --no-compare --no-e2e --no-cpu >> gpurun_out/g1_bench.jsonl 2>> gpurun_out/g1_bench.err
done
