mkdir -p gpurun_out
for v in default t1024 t1024b t4096; do
  echo "== $v"
  if [ $v = default ]; then unset SUNFOLD_LIB; else export SUNFOLD_LIB=$PWD/paper_1812_11626_b200/exp/libsunfold_$v.so; fi
  for c in 4 3; do timeout 300 python tools/time_apply.py $c 2>&1 | grep -v matrix-free; done
done > gpurun_out/ap_ab.log 2>&1
cat gpurun_out/ap_ab.log
