# round-2 final validation (4 GPUs) at HEAD c0bd01e: the driver's GPU suite, smoke, mp_worker logs, short bench lines
mkdir -p gpurun_out
echo "head c0bd01e" > gpurun_out/g28_head.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/g28_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g28_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g28_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/g28_smoke.log
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2966$n tests/mp_worker.py > gpurun_out/g28_multi_w$n.log 2>&1; echo "rc=$?" >> gpurun_out/g28_multi_w$n.log; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-compare --no-e2e --no-cpu > gpurun_out/g28_n1.json 2> gpurun_out/g28.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29777 bench.py --gpus 4 --steps 10 --warmup 3 --no-compare --no-e2e --no-cpu --nccl > gpurun_out/g28_n4.json 2>> gpurun_out/g28.err
