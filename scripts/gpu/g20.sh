# round-2 call (4 GPUs): HEAD f6b4632 -- full GPU suite (incl. multi-GPU), smoke, final bench lines, NVLS on P_k = 4 dims, N=1 ncu
mkdir -p gpurun_out
echo "head f6b4632" > gpurun_out/g20_head.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/g20_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g20_pytest.log
for n in 2 4; do timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n tests/mp_worker.py > gpurun_out/g20_multi_w$n.log 2>&1; echo "rc=$?" >> gpurun_out/g20_multi_w$n.log; done
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g20_smoke.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g20_n1.json 2> gpurun_out/g20.err
run() { timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $1 --steps 20 --warmup 5 "${@:2}"; }
run 2 > gpurun_out/g20_n2.json 2>> gpurun_out/g20.err
run 4 > gpurun_out/g20_n4.json 2>> gpurun_out/g20.err
run 4 --sizes 2,2 --ratio 1:1 --no-e2e --pace-gbs 660 > gpurun_out/g20_n4_2x2_p660.json 2>> gpurun_out/g20.err
run 4 --sizes 4 --ratio 1 --no-e2e --no-compare --nccl --nvls > gpurun_out/g20_n4_flat_nvls.json 2>> gpurun_out/g20.err
run 4 --sizes 4 --ratio 1 --no-e2e --no-compare --nccl > gpurun_out/g20_n4_flat.json 2>> gpurun_out/g20.err
run 4 --sizes 2,4 --ratio 1:1 --no-e2e --no-compare --nccl --nvls > gpurun_out/g20_n4_2x4_nvls.json 2>> gpurun_out/g20.err
B="python bench.py --steps 2 --warmup 3 --no-compare --no-e2e --no-cpu"
$B > gpurun_out/g20_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g20_launches.csv $B > /dev/null 2>> gpurun_out/g20.err && ncu --set full --import-source on --clock-control none -k regex:themis_exec -s 3 -c 1 -o gpurun_out/g20_full_n1 $B > /dev/null 2>> gpurun_out/g20.err
