# round-2 call 1 (4 GPUs): HEAD multi-GPU parity, NVLink engine probe, 4-GPU topologies
set -x
mkdir -p gpurun_out
echo "head 227d847" > gpurun_out/g2_head.txt
nvidia-smi topo -m > gpurun_out/g2_topo.txt 2>&1
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n tests/mp_worker.py > gpurun_out/g2_multi_w$n.log 2>&1; echo "rc=$?" >> gpurun_out/g2_multi_w$n.log; done
bash scripts/nvlink/sweep.sh $PWD/gpurun_out/g2_probe.jsonl > gpurun_out/g2_sweep.log 2>&1
for sz in "2,2 1:1" "4,2 1:1" "2,4 1:1"; do set -- $sz
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 10 --warmup 3 --sizes $1 --ratio $2 --no-e2e --no-cpu >> gpurun_out/g2_bench.jsonl 2>> gpurun_out/g2_bench.err
done
