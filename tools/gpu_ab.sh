# A/B of an env switch (AB_VAR, e.g. SUNFOLD_MODE2=1) on config CFG: GPU tests (PYTEST_SEL), bench lines
# with and without the switch, launch lists of both
mkdir -p gpurun_out
CFG=${CFG:-3}
timeout 900 python -m pytest ${PYTEST_SEL:-tests -m gpu} -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/ab_pytest.log
timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/ab_bench_new.log 2>&1; echo bench_new=$?
env $AB_VAR timeout 300 python bench.py --config $CFG --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/ab_bench_old.log 2>&1; echo bench_old=$?
python tools/prof_unfold.py --config $CFG --iters 5 --reuse-plan > /dev/null 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launches_new.csv python tools/prof_unfold.py --config $CFG --iters 5 --reuse-plan > /dev/null 2>&1; echo ncu_new=$?
env $AB_VAR timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_launches_old.csv python tools/prof_unfold.py --config $CFG --iters 5 --reuse-plan > /dev/null 2>&1; echo ncu_old=$?
