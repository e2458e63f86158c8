# Re-entry verification: full GPU tests, smoke, default bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/verify_pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/verify_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/verify_bench.log 2>gpurun_out/verify_bench.err; echo bench=$?
