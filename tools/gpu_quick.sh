# quick GPU iteration: selected GPU tests (PYTEST_SEL) and a c4 bench line (BENCH_ARGS)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest ${PYTEST_SEL:-tests -m gpu} -x -q > gpurun_out/pytest_quick.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_quick.log
timeout 600 python bench.py ${BENCH_ARGS:---no-cpu-baseline --no-e2e --no-rk4 --no-f3} > gpurun_out/bench_quick.log 2>&1; echo bench=$?
tail -c 600 gpurun_out/bench_quick.log
