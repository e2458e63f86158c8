"""Time sun_apply (dv/dt = Q0 v + eps Q1 v + K) at a BASELINE config (L2 flushed before each call)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_11626_b200 as sun  # noqa: E402
from workloads import config  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 4
p = config(idx)
Q0, Q1, K = sun.unfold(p.H0, p.H1, p.Ls, p.gammas)
v = torch.randn(Q0.m, dtype=torch.float64, device="cuda")
y = torch.empty_like(v)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
ts = []
for i in range(12):
    flush.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sun.apply(Q0, Q1, 1.3, K, v, out=y)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts = sorted(ts[2:])
nz = Q0.nnz + (Q1.nnz if Q1 is not None else 0)
byts = 12 * nz + 8 * (Q0.m + 1) * (2 if Q1 is not None else 1) + 8 * Q0.m * 3
print(f"config {idx} apply {ts[len(ts)//2]*1e3:.1f} us, {byts / (ts[len(ts)//2]*1e-3) / 1e9:.0f} GB/s algorithmic")
# matrix-free (sun_apply_plan) on the plan of the same problem
plan = sun.Plan(p.H0, p.H1, p.Ls, p.gammas)
plan.run()
tm = []
for i in range(12):
    flush.fill_(1.0)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    plan.apply(v, 1.3, out=y)
    b.record()
    torch.cuda.synchronize()
    tm.append(a.elapsed_time(b))
tm = sorted(tm[2:])
print(f"config {idx} apply matrix-free {tm[len(tm)//2]*1e3:.1f} us")
