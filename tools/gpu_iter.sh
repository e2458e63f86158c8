# iteration: path diff, quick bench, launch list of a few plan.run() calls
mkdir -p gpurun_out
timeout 300 python tools/diff_paths.py ${DIFFVAR:-SUNFOLD_NO_PROLOGUE=1} > gpurun_out/diff.log 2>&1; echo diff=$?; tail -1 gpurun_out/diff.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-rk4 --no-f3 ${BENCH_ARGS:-} > gpurun_out/bench_quick.log 2>&1; echo bench=$?
python tools/prof_unfold.py --config ${CFG:-4} --iters 5 --reuse-plan > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/iter_launches.csv python tools/prof_unfold.py --config ${CFG:-4} --iters 5 --reuse-plan > /dev/null 2>&1; echo ncu=$?
