# ncu --set full with source counters of the fill kernel at c4 (one launch), after a plain run
mkdir -p gpurun_out
python tools/prof_unfold.py --config ${CFG:-4} --iters 3 --reuse-plan > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_fill0} -s ${SKIP:-1} -c 1 \
  -o gpurun_out/${OUT:-fill_full} -f python tools/prof_unfold.py --config ${CFG:-4} --iters 3 --reuse-plan > gpurun_out/ncu_fill.log 2>&1; echo ncu=$?
