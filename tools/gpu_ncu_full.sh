# one ncu --set full capture of the unfold kernels at c4 (after a plain run of the same command)
set -x
mkdir -p gpurun_out
CMD="python tools/prof_unfold.py --config ${CFG:-4} --iters 3 --reuse-plan"
$CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_fill|k_count|k_scan}" -s ${SKIP:-10} -c ${COUNT:-10} \
  -o gpurun_out/${OUT:-prof_full} -f $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
