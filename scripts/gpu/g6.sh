# round-2 call (4 GPUs): K5 over NVLink (one dim group alone, real executor, faked peer) + ncu NVLink counters
mkdir -p gpurun_out
K="python scripts/k5_nvlink.py --mib 512"
M="gpu__time_duration.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum"
pts=(
 "caps16 --ctas 16"
 "caps32 --ctas 32"
 "caps64 --ctas 64"
 "caps128 --ctas 128"
 "p421_d1 --ctas 73 --bw-gbs 411 --paced"
 "p421_d2 --ctas 37 --bw-gbs 206 --paced"
 "p421_d3 --ctas 18 --bw-gbs 103 --paced"
 "p111 --ctas 43 --bw-gbs 240 --paced"
 "p111n4 --ctas 32 --bw-gbs 160 --paced"
 "p421n4_d2 --ctas 43 --bw-gbs 160 --paced"
 "p421n4_d3 --ctas 21 --bw-gbs 80 --paced"
)
for pt in "${pts[@]}"; do set -- $pt; tag=$1; shift
  timeout 120 $K --tag $tag "$@" >> gpurun_out/g6_k5.jsonl 2>> gpurun_out/g6_k5.err && \
  timeout 300 ncu --metrics $M --clock-control none -k regex:themis_exec -s 2 -c 1 --csv --log-file gpurun_out/g6_ncu_$tag.csv $K --iters 1 --tag $tag "$@" > /dev/null 2>> gpurun_out/g6_ncu.err
done
# the all-NVLink 2x2 kernel of GPU 0 alone (3 faked peers): plain, then one full ncu capture
timeout 120 python scripts/k5_nvlink.py --sizes 2,2 --ctas 64,64 --bw-gbs 1,1 --mib 1024 --tag solo2x2 >> gpurun_out/g6_k5.jsonl 2>> gpurun_out/g6_k5.err
timeout 120 python scripts/k5_nvlink.py --sizes 2,2 --ctas 64,64 --bw-gbs 1,1 --mib 1024 --lookahead 16 --tag solo2x2_la16 >> gpurun_out/g6_k5.jsonl 2>> gpurun_out/g6_k5.err && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:themis_exec -s 2 -c 1 -o gpurun_out/g6_solo2x2 python scripts/k5_nvlink.py --sizes 2,2 --ctas 64,64 --bw-gbs 1,1 --mib 1024 --lookahead 16 --iters 1 > /dev/null 2>> gpurun_out/g6_ncu.err
