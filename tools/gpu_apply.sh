# streamed k_apply: GPU tests that use sun_apply, then its time at c4, c3, c2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_propagate.py tests/test_gpu_general.py tests/test_abi.py -x -q -m gpu > gpurun_out/ap_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ap_pytest.log
for c in 4 3 2; do timeout 300 python tools/time_apply.py $c; done > gpurun_out/ap_time.log 2>&1
cat gpurun_out/ap_time.log
