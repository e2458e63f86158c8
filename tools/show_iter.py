"""Print the quick-iteration results (gpurun_out/bench_quick.log, iter_launches.csv)."""
import csv
import json

l = [x for x in open('gpurun_out/bench_quick.log') if x.startswith('{')]
if l:
    d = json.loads(l[-1])
    print("c4", d['value'], d['ms_per_step'], "cold", d['unfold_cold_ms'], "fill frac", d['roofline']['frac'],
          d['phases_ms'], "oracle", d['oracle_check'] and d['oracle_check']['pattern_exact'])
    for k, v in d.get('configs', {}).items():
        print(" ", k, v['ms_per_step'], v['fill']['frac'], v['oracle_check']['pattern_exact'])
    for k, v in d.get('general_pattern', {}).items():
        print(" ", k, v['ms_per_step'], v['fill']['launch_ms'], v['oracle_check']['pattern_exact'])
else:
    print(open('gpurun_out/bench_quick.log').read()[-3000:])
try:
    rows = list(csv.reader(open('gpurun_out/iter_launches.csv')))
    i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[i]
    for r in rows[i + 1:]:
        if len(r) > 5 and r[h.index('Metric Name')] == 'gpu__time_duration.sum':
            print("  ", r[h.index('Kernel Name')][:60], r[h.index('Metric Value')])
except Exception as e:
    print("no launch list", e)
