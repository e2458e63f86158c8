"""Phases of a one-shot sun.unfold() at c4 (host wall clock, synchronised): plan creation, first
run, close; with outputs kept alive (fresh allocations) or released (allocator cache hits)."""
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1812_11626_b200 as sun  # noqa: E402
from workloads import config  # noqa: E402

prob = config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
H0 = sun.DeviceZCSR.from_host(prob.H0)
H1 = sun.DeviceZCSR.from_host(prob.H1) if prob.H1 is not None else None
Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
torch.cuda.synchronize()


def phases(keep):
    t0 = time.perf_counter()
    plan = sun.Plan(H0, H1, Ls, prob.gammas)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    out = plan.run()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    plan.close()
    t3 = time.perf_counter()
    if keep is not None:
        keep.append(out)
    return (t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3


for label, keep in (("outputs released", None), ("outputs kept", [])):
    for i in range(6):
        c, r, d = phases(keep)
        print(f"{label:17s} iter {i}: create {c:.3f} ms  first run {r:.3f} ms  close {d:.3f} ms  total {c + r + d:.3f}")
