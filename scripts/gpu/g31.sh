# round-2 last call (4 GPUs) at HEAD dc771da: GPU suite, smoke, full bench lines N=1 and N=4
mkdir -p gpurun_out
echo "head dc771da" > gpurun_out/g31_head.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/g31_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g31_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g31_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g31_n1.json 2> gpurun_out/g31.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29788 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/g31_n4.json 2>> gpurun_out/g31.err
