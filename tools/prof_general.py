"""Run the general-pattern unfold of one workload a few times with graphs off (for ncu launch lists)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1812_11626_b200 as sun  # noqa: E402
from workloads import dense_dissipator_problem, random_sparse_problem, ring_dimer_problem  # noqa: E402

W = {"sparse300": lambda: random_sparse_problem(300, seed=21, P=2), "ring1000": lambda: ring_dimer_problem(1000, True),
     "dense48": lambda: dense_dissipator_problem(48, seed=0), "sparse1000": lambda: random_sparse_problem(1000, seed=22, P=2)}
prob = W[sys.argv[1]]()
plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
plan.set_graphs(False)
for _ in range(2):
    plan.run()
torch.cuda.synchronize()
print("ok")
