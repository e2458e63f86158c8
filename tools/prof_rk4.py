"""Minimal driver for ncu: a few RK4 steps (sun_rk4) of the c4 system."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1812_11626_b200 as sun
    from workloads import ZCSR, config

    prob = config(4)
    Q0, Q1, K = sun.unfold(prob.H0, prob.H1, prob.Ls, prob.gammas)
    v = sun.expand_state(ZCSR.from_triplets(prob.n, [0], [0], [1.0]))
    sun.rk4(Q0, Q1, K, v, 1e-5, 2, eps0=1.0, eps1=1.5)
    torch.cuda.synchronize()
    print("ok", float(v.abs().max()))


if __name__ == "__main__":
    main()
