# round-2 call (4 GPUs): two-pass LL (R31) -- parity at N=1 / W=4 and latency-regime throughput
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_emulated.py -x -q -k "ll" > gpurun_out/g24_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g24_pytest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29654 tests/mp_worker.py > gpurun_out/g24_multi_w4.log 2>&1; echo "rc=$?" >> gpurun_out/g24_multi_w4.log
run() { timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu --no-compare "$@" 2>> gpurun_out/g24.err | tail -1; }
for mib in 1 4 16 64; do for sz in "2,2,2 4:2:1" "2,2 1:1"; do set -- $sz; for ch in 8 64; do
  echo "{\"mib\":$mib,\"sizes\":\"$1\",\"chunks\":$ch,\"ll\":256,\"line\":$(run --sizes $1 --ratio $2 --mib $mib --chunks $ch --ll-max-mib 256)}" >> gpurun_out/g24.jsonl
done; done; done
