"""Time the CSR and the matrix-free RK4 step on configs[3] (mode 2)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_11626_b200 as sun  # noqa: E402
from workloads import ZCSR, config  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = config(idx)
plan = sun.Plan(p.H0, p.H1, p.Ls, p.gammas)
Q0, Q1, K = plan.run()
v = sun.expand_state(ZCSR.from_triplets(p.n, [0], [0], [1.0]))
for name, fn in (("csr", lambda n: sun.rk4(Q0, Q1, K, v, 1e-5, n, eps0=1.0, eps1=1.5)),
                 ("mf", lambda n: plan.rk4(v, 1e-5, n, eps0=1.0, eps1=1.5))):
    fn(2)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn(20)
    b.record()
    torch.cuda.synchronize()
    print(f"config {idx} {name} {a.elapsed_time(b) / 20:.4f} ms/step")
