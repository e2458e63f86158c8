# bench line of config CFG under each env setting in ENVS (space-separated, "-" = none), REPS times, interleaved
mkdir -p gpurun_out
for r in $(seq ${REPS:-2}); do for e in ${ENVS}; do
  if [ "$e" = "-" ]; then E=; else E="$e"; fi
  env $E timeout 300 python bench.py --config ${CFG:-4} --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/eb.log 2>&1
  python -c "import json; d=json.loads([l for l in open('gpurun_out/eb.log') if l.startswith('{')][-1]); print('c${CFG:-4} $e', round(d['ms_per_step']*1e3,1), 'us fill', round(d['roofline']['launch_ms']*1e3,1), {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})"
done; done
