# round-2 call (4 GPUs): push-mode AG (R30): parity at N=1 and in the multi-GPU worker, then throughput
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "push or runtime or random_executor or watchdog" > gpurun_out/g12_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g12_pytest.log
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n tests/mp_worker.py > gpurun_out/g12_multi_w$n.log 2>&1; echo "rc=$?" >> gpurun_out/g12_multi_w$n.log; done
K="timeout 180 python scripts/k5_nvlink.py --sizes 2,2 --mib 1024 --bw-gbs 1,1 --ctas 64,64 --lookahead 16"
for pu in 0 1; do
  THEMIS_PUSH=$pu $K --all-gpus --tag all_push$pu >> gpurun_out/g12_k5.jsonl 2>> gpurun_out/g12.err
  THEMIS_PUSH=$pu $K --tag solo_push$pu >> gpurun_out/g12_k5.jsonl 2>> gpurun_out/g12.err
done
run() { timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --steps 10 --warmup 3 --no-e2e --no-cpu --no-compare --nccl "$@" 2>>gpurun_out/g12.err | tail -1; }
for pu in 0 1; do for sz in "2,2 1:1" "2,4 1:1" "2,2,2 4:2:1"; do set -- $sz
  echo "{\"push\":$pu,\"sizes\":\"$1\",\"line\":$(THEMIS_PUSH=$pu run --sizes $1 --ratio $2)}" >> gpurun_out/g12_bench.jsonl
done; done
