# round-2 call (4 GPUs): LL small collectives (R31) -- parity at N=1 and W=2/4, then latency-regime throughput
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_emulated.py -x -q -k "ll or watchdog or random" > gpurun_out/g23_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g23_pytest.log
for n in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n tests/mp_worker.py > gpurun_out/g23_multi_w$n.log 2>&1; echo "rc=$?" >> gpurun_out/g23_multi_w$n.log; done
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-cpu --no-compare --nccl "$@" 2>> gpurun_out/g23.err | tail -1; }
for mib in 1 4 16 64; do for sz in "2,2,2 4:2:1" "2,2 1:1"; do set -- $sz; for ch in 64 8; do for ll in 0 256; do
  echo "{\"mib\":$mib,\"sizes\":\"$1\",\"chunks\":$ch,\"ll\":$ll,\"line\":$(run --sizes $1 --ratio $2 --mib $mib --chunks $ch --ll-max-mib $ll)}" >> gpurun_out/g23.jsonl
done; done; done; done
