# round-2 call (4 GPUs): pipelined push AG vs pull, ring depth; push parity re-check
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulated.py -x -q -k "push" > gpurun_out/g14_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g14_pytest.log
K="timeout 180 python scripts/k5_nvlink.py --sizes 2,2 --mib 1024 --bw-gbs 1,1 --ctas 64,64 --lookahead 16 --all-gpus"
for pu in 0 1; do for st in "2 32" "3 32" "4 32" "3 48"; do set -- $st
  THEMIS_PUSH=$pu $K --stages $1 --stage-kb $2 --tag all_push${pu}_s$1_kb$2 >> gpurun_out/g14_k5.jsonl 2>> gpurun_out/g14.err
done; done
