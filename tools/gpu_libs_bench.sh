# bench line (ms per unfold, fill bracket) of each config in CFGS for the default lib and each exp lib in LIBS
mkdir -p gpurun_out
for c in ${CFGS:-4}; do for l in default ${LIBS}; do
  if [ $l = default ]; then E=; else E=SUNFOLD_LIB=paper_1812_11626_b200/exp/libsunfold_$l.so; fi
  env $E timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/lb_${l}_c$c.log 2>&1
  python -c "import json,sys; d=json.loads([l for l in open('gpurun_out/lb_${l}_c$c.log') if l.startswith('{')][-1]); print('c$c $l', round(d['ms_per_step']*1e3,1), 'us', 'fill', round(d['roofline']['launch_ms']*1e3,1), {k: round(v*1e3,1) for k,v in d['phases_ms'].items()})"
done; done
