"""Diagnostics: dense unfold vs oracle O3 at small N (prints the difference matrix)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1812_11626_b200 as sun
from oracle import gks
from workloads import gks_ensemble

np.set_printoptions(precision=3, suppress=True, linewidth=200)
for n in (2, 3):
    H, A = gks_ensemble(n, 1, seed=100 + n)
    dev = lambda x: torch.as_tensor(x).cuda()  # noqa: E731
    for a in (A, None):
        Q, K = sun.unfold_dense(dev(H), dev(a) if a is not None else None)
        torch.cuda.synchronize()
        Qo, Ko = gks.unfold_gks(H[0], a[0] if a is not None else None)
        D = Q.cpu().numpy()[0] - Qo
        print(n, 'A' if a is not None else 'noA', 'maxerr', np.abs(D).max())
        if np.abs(D).max() > 1e-9:
            print(np.round(D, 3))
