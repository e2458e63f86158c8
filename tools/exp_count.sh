# time count/fill of experiment builds (paper_1812_11626_b200/exp/libsunfold_*.so) at the given configs
mkdir -p gpurun_out
for f in paper_1812_11626_b200/exp/libsunfold_*.so; do
  for c in ${CFGS:-4}; do
    SUNFOLD_LIB=$f timeout 120 python tools/exp_fill.py $c
    SUNFOLD_LIB=$f timeout 120 python tools/timeline.py $c 2>/dev/null | grep -E "^  \+" | tail -4
  done
done
