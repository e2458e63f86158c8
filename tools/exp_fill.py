"""Time the fill pass (sun_unfold) and the count pass in isolation for the library named by
SUNFOLD_LIB (diagnostics: experiment builds with parts of the fill switched off)."""
import os
import statistics
import sys

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
    plan.count()
    n0, n1 = plan.nnz()
    outs = plan.fill(n0, n1)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    res = {}
    def count():
        plan.count()
        plan.nnz()

    for name, fn in (("count+nnz", count), ("fill", lambda: plan.fill(n0, n1, out=outs))):
        ts = []
        for i in range(25):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        d = [a.elapsed_time(b) * 1e3 for a, b in ts[5:]]
        res[name] = statistics.median(d)
    print(os.path.basename(os.environ.get("SUNFOLD_LIB", "default")), {k: round(v, 1) for k, v in res.items()}, "us")


if __name__ == "__main__":
    main()
