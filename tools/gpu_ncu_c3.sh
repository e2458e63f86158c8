# c3: bench with/without near_sep, launch list with near_sep, ncu --set full of fill/near/count
mkdir -p gpurun_out
timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/c3_bench_a.log 2>&1; echo a=$?
SUNFOLD_NEAR_SEP=1 timeout 300 python bench.py --config 3 --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/c3_bench_b.log 2>&1; echo b=$?
SUNFOLD_NEAR_SEP=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_launches_b.csv python tools/prof_unfold.py --config 3 --iters 5 --reuse-plan > /dev/null 2>&1; echo ncu_b=$?
SUNFOLD_NEAR_SEP=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fill0|k_count0|k_near0" -s 3 -c 3 \
  -o gpurun_out/c3_full -f python tools/prof_unfold.py --config 3 --iters 3 --reuse-plan > gpurun_out/c3_ncu.log 2>&1; echo ncufull=$?
