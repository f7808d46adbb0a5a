# round-2 call (1 GPU): LL after the CTA-uniform go/abort fix -- watchdog + LL tests with per-test timeouts
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_emulated.py -v -x --timeout 120 -k "ll_small or ll_falls or watchdog" > gpurun_out/g26_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/g26_pytest.log
