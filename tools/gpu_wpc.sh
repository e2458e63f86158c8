# count pass: warps (units) per CTA, A/B through SUNFOLD_LIB builds; bench lines at c4 and c3, interleaved twice
mkdir -p gpurun_out
B="--no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs"
for r in 1 2; do for c in 4 3; do for v in default wpc2 wpc4; do
  if [ $v = default ]; then unset SUNFOLD_LIB; else export SUNFOLD_LIB=$PWD/paper_1812_11626_b200/exp/libsunfold_$v.so; fi
  timeout 300 python bench.py --config $c $B > gpurun_out/wpc_${v}_c${c}_$r.log 2>&1; echo $v $c $?
done; done; done
