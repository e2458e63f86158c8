"""Per-step timing of plan.run() under the bench's conditions, one factor at a time (diagnostics):
plain / + L2 flush / + keeping outputs alive / + nvidia-smi clock sampler."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    import paper_1812_11626_b200 as sun
    from workloads import config

    prob = config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
    H0 = sun.DeviceZCSR.from_host(prob.H0)
    H1 = sun.DeviceZCSR.from_host(prob.H1) if prob.H1 is not None else None
    Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
    plan = sun.Plan(H0, H1, Ls, prob.gammas)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(5):
        plan.run()
    torch.cuda.synchronize()

    def loop(n, do_flush, keep_n, sampler):
        keep, ev, host = [], [], []
        ctx = bench.ClockSampler(0) if sampler else None
        if ctx:
            ctx.__enter__()
        for _ in range(n):
            if do_flush:
                flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            out = plan.run()
            e1.record(stream)
            host.append((time.perf_counter() - t0) * 1e3)
            ev.append((e0, e1))
            if keep_n:
                keep.append(out)
                if len(keep) > keep_n:
                    keep.pop(0)
        torch.cuda.synchronize()
        if ctx:
            ctx.__exit__(None, None, None)
        d = [a.elapsed_time(b) for a, b in ev]
        return d, host

    for name, kw in [("plain", dict(do_flush=False, keep_n=0, sampler=False)),
                     ("flush", dict(do_flush=True, keep_n=0, sampler=False)),
                     ("flush+keep2", dict(do_flush=True, keep_n=2, sampler=False)),
                     ("flush+keep2+sampler", dict(do_flush=True, keep_n=2, sampler=True)),
                     ("plain again", dict(do_flush=False, keep_n=0, sampler=False))]:
        d, h = loop(40, **kw)
        print(f"{name:22s} device ms: median {statistics.median(d):.4f} mean {statistics.mean(d):.4f} "
              f"max {max(d):.4f} | host ms: median {statistics.median(h):.4f} max {max(h):.4f}")


if __name__ == "__main__":
    main()
