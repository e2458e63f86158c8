# A/B of the fused scan + near rows launch (k_scan_near0; SUNFOLD_SCAN_NEAR=0: scan then k_near0 / near units
# inside the fill) at c4 and c3: GPU tests, bench lines (interleaved twice), launch lists
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guards.py tests/test_gpu_propagate.py -x -q > gpurun_out/sn_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/sn_pytest.log
B="--no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs"
for r in 1 2; do
for c in 4 3; do
timeout 300 python bench.py --config $c $B > gpurun_out/sn_bench_c${c}_new$r.log 2>&1; echo bench_new$c=$?
SUNFOLD_SCAN_NEAR=0 timeout 300 python bench.py --config $c $B > gpurun_out/sn_bench_c${c}_old$r.log 2>&1; echo bench_old$c=$?
done; done
for c in 4 3; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sn_launches_c${c}_new.csv python tools/prof_unfold.py --config $c --iters 5 --reuse-plan > /dev/null 2>&1; echo ncu_new=$?
SUNFOLD_SCAN_NEAR=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sn_launches_c${c}_old.csv python tools/prof_unfold.py --config $c --iters 5 --reuse-plan > /dev/null 2>&1; echo ncu_old=$?
done
