"""Instruction mix (warp-level executed instructions per SASS opcode) from an
`ncu --page source --csv --print-source cuda,sass` (or sass) export."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
mix = collections.Counter()
h = None
for r in rows:
    if r and r[0] in ('Line No', 'Address'):
        h = r
        continue
    if h is None or len(r) < 8:
        continue
    if h[0] == 'Line No':
        if r[0] != '' or len(r) < 8:
            continue
        src, cnt = r[3], r[7]
    else:
        src, cnt = r[1], r[5]
    try:
        n = int(cnt or 0)
    except ValueError:
        continue
    m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?', src)
    if m:
        mix[m.group(2) + (m.group(3) or '')[:12]] += n
tot = sum(mix.values())
print('total', tot)
for k, v in mix.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    print(f"{v:11d} {100.0 * v / tot:5.1f}% {k}")
