"""Measure host-side (Python + C-ABI) overhead of each phase of an unfold (diagnostics)."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1812_11626_b200 as sun
    from workloads import config

    prob = config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
    H0 = sun.DeviceZCSR.from_host(prob.H0)
    H1 = sun.DeviceZCSR.from_host(prob.H1) if prob.H1 is not None else None
    Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
    plan = sun.Plan(H0, H1, Ls, prob.gammas)
    rec = {k: [] for k in ("plan_create", "count_call", "nnz_call", "fill_call", "sync_after_fill", "empty3", "close")}
    for it in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p2 = sun.Plan(H0, H1, Ls, prob.gammas)
        t1 = time.perf_counter()
        p2.close()
        t2 = time.perf_counter()
        plan.count()
        t3 = time.perf_counter()
        n0, n1 = plan.nnz()
        t4 = time.perf_counter()
        out = plan.fill(n0, n1)
        t5 = time.perf_counter()
        torch.cuda.synchronize()
        t6 = time.perf_counter()
        a = torch.empty(2 * (prob.m + 1), dtype=torch.int64, device="cuda")
        b = torch.empty(n0 + n1, dtype=torch.int32, device="cuda")
        c = torch.empty(n0 + n1 + prob.m, dtype=torch.float64, device="cuda")
        t7 = time.perf_counter()
        del a, b, c
        if it >= 5:
            rec["plan_create"].append(t1 - t0)
            rec["close"].append(t2 - t1)
            rec["count_call"].append(t3 - t2)
            rec["nnz_call"].append(t4 - t3)
            rec["fill_call"].append(t5 - t4)
            rec["sync_after_fill"].append(t6 - t5)
            rec["empty3"].append(t7 - t6)
    for k, v in rec.items():
        print(f"{k:18s} median {statistics.median(v) * 1e6:9.1f} us")


if __name__ == "__main__":
    main()
