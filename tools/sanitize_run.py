"""Small end-to-end run of every device entry point (for compute-sanitizer): unfold (graph and
direct), two-pass API, apply, expand_state, state_diag, rk4 on configs[0..2] + a mode-1 case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1812_11626_b200 as sun
    from workloads import ZCSR, banded_random_problem, config

    probs = [config(0), config(1), config(2), banded_random_problem(40, seed=3)]
    for prob in probs:
        plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
        Q0, Q1, K = plan.run()
        plan.set_graphs(False)
        Q0, Q1, K = plan.run_two_pass()
        v = sun.expand_state(ZCSR.from_triplets(prob.n, [0], [0], [1.0]))
        y = sun.apply(Q0, Q1, 1.0, K, v)
        sun.rk4(Q0, Q1, K, v, 1e-4, 3, eps0=1.0, eps1=1.5)
        d = sun.state_diag(v, prob.n)
        torch.cuda.synchronize()
        print(prob.name, Q0.nnz, float(d.sum()), float(y.abs().max()))
        plan.close()


if __name__ == "__main__":
    main()
