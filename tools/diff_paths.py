"""Diagnostics: plan.run() with the default launch structure against a plan created with the
environment variable given in argv[1] set (e.g. SUNFOLD_NO_PROLOGUE=1): first differing rows."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_11626_b200 as sun
from workloads import banded_random_problem, config, dimer_problem


def cmp(name, a, b):
    ra, rb = a.row_ptr.cpu().numpy(), b.row_ptr.cpu().numpy()
    bad = np.nonzero(ra != rb)[0]
    msg = f"  {name}: nnz {a.nnz} vs {b.nnz}; row_ptr diffs {bad.size}"
    if bad.size:
        msg += f" first at row {bad[0]}: {ra[bad[0]]} vs {rb[bad[0]]}"
    else:
        va, vb = a.val.cpu().numpy(), b.val.cpu().numpy()
        d = np.nonzero((a.col.cpu().numpy() != b.col.cpu().numpy()) | (va != vb))[0]
        rel = np.abs(va - vb).max() / max(np.abs(vb).max(), 1e-300) if va.size else 0.0
        msg += f"; entry diffs {d.size}" + (f" first at {d[0]}, max rel {rel:.2e}" if d.size else "")
    print(msg, flush=True)
    return bad.size == 0


var, val = (sys.argv[1].split("=") + ["1"])[:2] if len(sys.argv) > 1 else ("SUNFOLD_NO_PROLOGUE", "1")
ok = True
for prob in [dimer_problem(2, True), dimer_problem(5, True), dimer_problem(16, False), dimer_problem(16, True),
             dimer_problem(130, True), config(1), config(2), config(4), dimer_problem(1300, True),
             banded_random_problem(300, seed=14, wH=2, wL=0, P=0), banded_random_problem(77, seed=13, wH=1, wL=1, P=2),
             banded_random_problem(257, seed=15, wH=1, wL=0, P=3), banded_random_problem(45, seed=12, wH=3, wL=0, P=1)]:
    os.environ.pop(var, None)
    pa = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    os.environ[var] = val
    pb = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    os.environ.pop(var, None)
    ia, ib = pa.info(), pb.info()
    a = [pa.run(), pa.run(), pa.run_two_pass()]
    b = pb.run()
    torch.cuda.synchronize()
    print(prob.name, "launches", ia["launches_count"], ib["launches_count"], flush=True)
    for k, x in enumerate(a):
        ok &= cmp(f"Q0[{k}]", x[0], b[0])
        if x[1] is not None:
            ok &= cmp(f"Q1[{k}]", x[1], b[1])
        ok &= bool(torch.equal(x[2], b[2]))
    pa.close()
    pb.close()
print("ALL_EQUAL" if ok else "DIFFER")
