# A/B of an env switch (AB_VAR) on the bench line of each config in CFGS (after the GPU tests, PYTEST_SEL)
mkdir -p gpurun_out
timeout 900 python -m pytest ${PYTEST_SEL:-tests -m gpu} -x -q > gpurun_out/ab_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/ab_pytest.log
for c in ${CFGS:-4 3}; do for v in new old; do
  if [ $v = old ]; then E="$AB_VAR"; else E=""; fi
  env $E timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-rk4 --no-f3 --no-configs > gpurun_out/ab_${v}_c$c.log 2>&1
  python -c "import json,sys; d=json.loads([l for l in open('gpurun_out/ab_${v}_c$c.log') if l.startswith('{')][-1]); print('c$c $v', round(d['ms_per_step']*1e3,1), 'us', d['value'], 'fill', round(d['roofline']['launch_ms']*1e3,1), d['phases_ms'])"
done; done
