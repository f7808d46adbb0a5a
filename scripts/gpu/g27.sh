# round-2 call (1 GPU): LL watchdog after the uniform-exit fix
mkdir -p gpurun_out
timeout 420 python -m pytest tests/test_gpu_emulated.py -v -x --timeout 120 -k "ll_small or ll_falls or watchdog" > gpurun_out/g27_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g27_pytest.log
