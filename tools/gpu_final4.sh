# final state check: full GPU tests, smoke, default bench line, launch list of the same command
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/final_bench.log 2>gpurun_out/final_bench.err; echo bench=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-f3 --no-configs > /dev/null 2>&1; echo launches=$?
