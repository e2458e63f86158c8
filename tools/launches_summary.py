"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list (per kernel: launches, mean, share)."""
import collections
import csv
import sys


def main(path, title=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    ours = {k: v for k, v in d.items() if not k.startswith("void at::")}
    tot = sum(sum(v) for v in ours.values())
    out = []
    if title:
        out.append("# " + title)
    out.append("# per-launch device time in ns (cold-cache, serialised by ncu: compare shares, not absolutes)")
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        s = f" share_of_ours={sum(v) / tot:.3f}" if k in ours else ""
        out.append(f"{k:45s} launches={len(v):3d} mean_ns={sum(v) / len(v):10.1f} total_ns={sum(v):11.1f}{s}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
