# per-kernel launch list (ncu gpu__time_duration) of config CFG for the default lib and each exp lib in LIBS
mkdir -p gpurun_out
python tools/prof_unfold.py --config ${CFG:-4} --iters 5 --reuse-plan > /dev/null 2>&1
for l in default ${LIBS}; do
  if [ $l = default ]; then E=; else E=SUNFOLD_LIB=paper_1812_11626_b200/exp/libsunfold_$l.so; fi
  env $E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$l.csv python tools/prof_unfold.py --config ${CFG:-4} --iters 5 --reuse-plan > /dev/null 2>&1
  echo "== $l"; python tools/launches_summary.py gpurun_out/ll_$l.csv | grep -v "^#"
done
