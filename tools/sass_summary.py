"""SASS evidence for the fill / general kernels: counts of TMA bulk copies (UBLKCP), async-proxy
fences and fp64 instructions per kernel, from cuobjdump -sass of the built libsunfold.so.
Usage: python tools/sass_summary.py > profiles/rNN_sass_summary.txt"""
import collections
import os
import re
import subprocess
import sys

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1812_11626_b200", "libsunfold.so")
sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1] if len(sys.argv) > 1 else LIB], capture_output=True,
                      text=True).stdout
cur, cnt = None, collections.OrderedDict()
OPS = ("UBLKCP", "UTMASTG", "UTMALDG", "FENCE.VIEW.ASYNC", "DFMA", "DADD", "DMUL", "SHFL", "BAR.SYNC")
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        cnt[cur] = collections.Counter()
        continue
    if cur:
        for op in OPS:
            if op in line:
                cnt[cur][op] += 1
print("kernel | " + " | ".join(OPS))
for f, c in cnt.items():
    dem = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
    print(f"{dem[:100]} | " + " | ".join(str(c.get(op, 0)) for op in OPS))
