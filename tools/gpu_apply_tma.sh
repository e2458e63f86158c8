# k_apply_tma (TMA bulk loads into a shared-memory ring) vs k_apply (register loads): tests, then times
mkdir -p gpurun_out
timeout 120 python tools/time_apply.py 2 > gpurun_out/tma_first.log 2>&1; echo first=$?; cat gpurun_out/tma_first.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_propagate.py tests/test_gpu_general.py tests/test_abi.py -x -q -m gpu -k "apply or abi or rk4 or general_patterns" > gpurun_out/tma_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/tma_pytest.log
for r in 1 2; do for v in 1 0; do for c in 4 3; do
  echo "== tma=$v c$c"; SUNFOLD_APPLY_TMA=$v timeout 120 python tools/time_apply.py $c 2>&1 | grep -v matrix-free
done; done; done > gpurun_out/tma_time.log 2>&1
cat gpurun_out/tma_time.log
