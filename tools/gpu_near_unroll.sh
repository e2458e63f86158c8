# k_near0 window-copy unroll (2 / 4 / 8 iterations' loads in flight) at c3: bench lines interleaved, launch lists
mkdir -p gpurun_out
B="--no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs"
for r in 1 2; do for v in default nu2 nu8; do
  if [ $v = default ]; then unset SUNFOLD_LIB; else export SUNFOLD_LIB=$PWD/paper_1812_11626_b200/exp/libsunfold_$v.so; fi
  timeout 300 python bench.py --config 3 $B > gpurun_out/nu_${v}_$r.log 2>&1; echo $v $?
done; done
for v in default nu2 nu8; do
  if [ $v = default ]; then unset SUNFOLD_LIB; else export SUNFOLD_LIB=$PWD/paper_1812_11626_b200/exp/libsunfold_$v.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:k_near0 --log-file gpurun_out/nu_launches_$v.csv python tools/prof_unfold.py --config 3 --iters 5 --reuse-plan > /dev/null 2>&1
done
