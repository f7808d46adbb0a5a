# round-2 call (4 GPUs): LL path out of line -- LL/watchdog tests + N=4 A/B vs f6b4632
mkdir -p gpurun_out
R=$PWD
timeout 300 python -m pytest tests/test_gpu_emulated.py -x -q --timeout 120 -k "ll_small or ll_falls or watchdog or runtime" > gpurun_out/g30_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g30_pytest.log
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-compare --no-e2e --no-cpu 2>/dev/null | tail -1; }
for rep in 1 2 3; do
  echo "{\"tag\":\"head_n4\",\"line\":$(run)}" >> gpurun_out/g30.jsonl
  echo "{\"tag\":\"old_n4\",\"line\":$(cd $R/old_f6b && run)}" >> gpurun_out/g30.jsonl
done
