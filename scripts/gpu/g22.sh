# round-2 call (1 GPU): randomised executor parity at scale (new paths: unit queue, runtime order, windows, push AG)
mkdir -p gpurun_out
for seed in 1 2 3; do
  THEMIS_RANDOM_SEED=$seed THEMIS_RANDOM_CASES=150 timeout 1200 python -m pytest tests/test_gpu_emulated.py -x -q -k "random_executor or random_rs_ag" > gpurun_out/g22_seed$seed.log 2>&1; echo "rc=$?" >> gpurun_out/g22_seed$seed.log
done
