# diagnostics: device timeline of a step, then one ncu --set full capture of the unfold kernels
set -x
mkdir -p gpurun_out
timeout 300 python tools/timeline.py 4 > gpurun_out/timeline.log 2>&1; echo timeline=$?
CMD="python tools/prof_unfold.py --config ${CFG:-4} --iters 3 --reuse-plan"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_fill|k_count|k_scan|k_expand}" -s ${SKIP:-7} -c ${COUNT:-7} \
  -o gpurun_out/${OUT:-prof_full} -f $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
