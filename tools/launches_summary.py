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
    def mine(k):  # this library's kernels (libsunfold.so): k_* names
        base = k.replace("void ", "").replace("<unnamed>", "").split("<")[0].split("::")[-1]
        return base.startswith("k_")

    ours = {k: v for k, v in d.items() if mine(k)}
    tot = sum(sum(v) for v in ours.values())
    step_names = ("k_expand", "k_count", "k_scan", "k_fill")  # one unfold step (sun_run)
    step = {k: v for k, v in ours.items() if any(n in k for n in step_names)}
    per_step = {k: sum(v) / len(v) for k, v in step.items()}
    step_tot = sum(per_step.values())
    out = []
    if title:
        out.append("# " + title)
    out.append("# per-launch device time in ns (cold-cache, serialised by ncu: compare shares, not absolutes)")
    out.append("# share_of_ours: of all libsunfold kernels in the run; share_of_step: mean launch time over the")
    out.append("# sum of the unfold step's kernels' mean launch times (expand + count + scan + fill)")
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        s = f" share_of_ours={sum(v) / tot:.3f}" if k in ours else " (not this library)"
        if k in per_step:
            s += f" share_of_step={per_step[k] / step_tot:.3f}"
        out.append(f"{k:45s} launches={len(v):3d} mean_ns={sum(v) / len(v):10.1f} total_ns={sum(v):11.1f}{s}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
