mkdir -p gpurun_out
for w in 1 2 4; do
  SUNFOLD_COUNT_WPC=$w timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_count0 --log-file gpurun_out/wpc_$w.csv python tools/prof_unfold.py --config 4 --iters 5 --reuse-plan > /dev/null 2>&1
  SUNFOLD_COUNT_WPC=$w timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/bench_wpc_$w.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_count0 -s 2 -c 1 -o gpurun_out/count_full -f python tools/prof_unfold.py --config 4 --iters 3 --reuse-plan > gpurun_out/ncu_count.log 2>&1; echo ncu=$?
