# general-pattern mode: GPU tests + bench lines of the general workloads
timeout 600 python -m pytest tests/test_gpu_general.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-rk4 --no-f3 > gpurun_out/gen.log 2>&1
tail -1 gpurun_out/gen.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d['general_pattern'].items(): print(k, round(v['ms_per_step'],4), '%.3g'%v['nnz_per_s'], 'fill', round(v['fill']['launch_ms'],4), v['oracle_check']['pattern_exact'], v['oracle_check']['max_err_normwise'])
"
