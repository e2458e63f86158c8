"""Per-source-line stall samples / instructions from an `ncu --page source --csv --print-source cuda,sass` export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, h, agg = None, None, {}
for r in rows:
    if len(r) == 2 and r[0] == 'File Name':
        fname = r[1].split('/')[-1]
        continue
    if r and r[0] == 'Line No':
        h = r
        continue
    if h is None or len(r) < 8 or r[0] == '':
        continue
    try:
        smp, ins = int(r[6] or 0), int(r[7] or 0)
    except ValueError:
        continue
    st = {}
    for k, name in enumerate(h):
        if name.startswith('stall_') and '(Not' not in name and k < len(r):
            try:
                v = int(r[k] or 0)
            except ValueError:
                v = 0
            if v:
                st[name[6:]] = v
    top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    agg[(fname, int(r[0]))] = (smp, ins, r[1].strip()[:70], top3)
tot = sum(v[0] for v in agg.values())
print('samples', tot, 'instructions', sum(v[1] for v in agg.values()))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:6d} {100.0 * v[0] / max(tot, 1):5.1f}% {v[1]:9d} {k[0]}:{k[1]} {v[2]}  {v[3]}")
