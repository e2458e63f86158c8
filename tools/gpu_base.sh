# session-start check: GPU tests, bench line with per-config lines, launch lists at c4 and c3
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/base_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/base_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-rk4 > gpurun_out/base_bench.log 2>&1; echo bench=$?
for c in 4 3; do
python tools/prof_unfold.py --config $c --iters 5 --reuse-plan > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/base_launches_c$c.csv python tools/prof_unfold.py --config $c --iters 5 --reuse-plan > /dev/null 2>&1; echo ncu$c=$?
done
