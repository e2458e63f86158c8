# A/B of env settings (each line of $ABFILE: "<cfg> <VAR=val,VAR=val|->"), REPS interleaved reps
mkdir -p gpurun_out
for r in $(seq ${REPS:-2}); do while read cfg e; do
  [ -z "$cfg" ] && continue
  if [ "$e" = "-" ]; then E=; else E="${e//,/ }"; fi
  env $E timeout 300 python bench.py --config $cfg --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/eb.log 2>&1
  python -c "import json; d=json.loads([l for l in open('gpurun_out/eb.log') if l.startswith('{')][-1]); print('c$cfg $e', round(d['ms_per_step']*1e3,1), 'us fill', round(d['roofline']['launch_ms']*1e3,1), 'frac', round(d['roofline']['frac'],3), {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})" || tail -5 gpurun_out/eb.log
done < ${ABFILE}; done
