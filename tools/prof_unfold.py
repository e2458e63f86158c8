"""Minimal driver for ncu / compute-sanitizer: run the unfold of one BASELINE config a few times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--reuse-plan", action="store_true")
    args = ap.parse_args()
    import torch

    import paper_1812_11626_b200 as sun
    from workloads import config

    prob = config(args.config)
    H0 = sun.DeviceZCSR.from_host(prob.H0)
    H1 = sun.DeviceZCSR.from_host(prob.H1) if prob.H1 is not None else None
    Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
    plan = sun.Plan(H0, H1, Ls, prob.gammas) if args.reuse_plan else None
    for _ in range(args.iters):
        if plan is None:
            Q0, Q1, K = sun.unfold(H0, H1, Ls, prob.gammas)
        else:
            Q0, Q1, K = plan.run()
    torch.cuda.synchronize()
    print("nnz", Q0.nnz, Q1.nnz if Q1 is not None else 0)


if __name__ == "__main__":
    main()
