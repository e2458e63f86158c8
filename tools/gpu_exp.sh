# experiment-lib A/B: tools/exp_fill.py (count / fill medians) for the default lib and each EXP_LIBS entry, on CFGS
mkdir -p gpurun_out
for c in ${CFGS:-3 4}; do
  timeout 120 python tools/exp_fill.py $c >> gpurun_out/exp.log 2>&1
  for l in ${EXP_LIBS}; do SUNFOLD_LIB=paper_1812_11626_b200/exp/libsunfold_$l.so timeout 120 python tools/exp_fill.py $c >> gpurun_out/exp.log 2>&1; done
done
cat gpurun_out/exp.log
