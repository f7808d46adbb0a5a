# round-2 call (4 GPUs): N=1 static vs runtime order, N=2/4 headline topology, N=1 ncu launch list + full capture
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 --lookahead 1 > gpurun_out/g10_n1_la1.json 2> gpurun_out/g10.err
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/g10_n1_la16.json 2>> gpurun_out/g10.err
run() { timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $1 --steps 20 --warmup 5 "${@:2}"; }
run 4 > gpurun_out/g10_n4.json 2>> gpurun_out/g10.err
run 2 > gpurun_out/g10_n2.json 2>> gpurun_out/g10.err
B="python bench.py --steps 2 --warmup 3 --no-compare --no-e2e --no-cpu"
$B > gpurun_out/g10_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/g10_launches.csv $B > /dev/null 2>> gpurun_out/g10.err && \
ncu --set full --import-source on --clock-control none -k regex:themis_exec -s 3 -c 1 -o gpurun_out/g10_full_n1 $B > /dev/null 2>> gpurun_out/g10.err
