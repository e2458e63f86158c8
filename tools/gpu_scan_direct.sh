# chain-free scan (every chunk's CTA sums the slots before it; SUNFOLD_SCAN_DIRECT=0: decoupled look-back chain):
# GPU tests, bench lines at c4, c3, c2 interleaved twice, launch lists
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_propagate.py -x -q > gpurun_out/sd_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/sd_pytest.log
B="--no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs"
for r in 1 2; do for c in 4 3 2; do for v in 1 0; do
  SUNFOLD_SCAN_DIRECT=$v timeout 300 python bench.py --config $c $B > gpurun_out/sd_bench_c${c}_v${v}_$r.log 2>&1; echo $c $v $?
done; done; done
for v in 1 0; do
SUNFOLD_SCAN_DIRECT=$v timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sd_launches_c4_v$v.csv python tools/prof_unfold.py --config 4 --iters 5 --reuse-plan > /dev/null 2>&1; echo ncu=$?
done
