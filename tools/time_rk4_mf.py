import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1812_11626_b200 as sun
from workloads import config, ZCSR
p = config(4)
plan = sun.Plan(p.H0, p.H1, p.Ls, p.gammas)
Q0, Q1, K = plan.run()
v = sun.expand_state(ZCSR.from_triplets(p.n, [0], [0], [1.0]))
w1 = torch.empty((int(sun.lib().sun_rk4_work_bytes(Q0.m)) + 7) // 8, dtype=torch.float64, device="cuda")
for name, fn in (("csr", lambda n: sun.rk4(Q0, Q1, K, v, 1e-5, n, eps0=1.0, eps1=1.5, work=w1)),
                 ("mf", lambda n: plan.rk4(v, 1e-5, n, eps0=1.0, eps1=1.5))):
    fn(2); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); fn(20); b.record(); torch.cuda.synchronize()
    print(name, a.elapsed_time(b) / 20, "ms/step")
