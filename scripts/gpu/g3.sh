# round-2 call (1 GPU): GPU suite + headline bench after the ADVICE fixes
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g3_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g3_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
python scripts/nvml_nvlink.py > gpurun_out/g3_nvml.txt 2>&1
