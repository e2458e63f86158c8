"""Unfold time vs Hilbert dimension N for the driven dimer (the paper's Figs. 4-7 axis):
one B200, device time per unfold (sun_run + nnz readback, CUDA events, L2 flushed), nnz/s,
fill-kernel GB/s; one JSON line per N."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1812_11626_b200 as sun
    from workloads import dimer_problem

    sizes = [int(x) for x in sys.argv[1:]] or [250, 500, 1000, 2000, 4000, 8000]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for n in sizes:
        prob = dimer_problem(n, True, name=f"dimer_N{n}_drive")
        H0 = sun.DeviceZCSR.from_host(prob.H0)
        H1 = sun.DeviceZCSR.from_host(prob.H1)
        Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
        plan = sun.Plan(H0, H1, Ls, prob.gammas)
        out = plan.run()
        nnz = out[0].nnz + out[1].nnz
        reps = 10 if n <= 2000 else 4
        ts = []
        for _ in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            out = plan.run(out=out)
            b.record(st)
            ts.append((a, b))
        torch.cuda.synchronize()
        ms = statistics.median(x.elapsed_time(y) for x, y in ts)
        # fill kernel alone (no graph replay)
        plan.set_graphs(False)
        plan.count()
        n0, n1 = plan.nnz()
        fs = []
        for _ in range(reps):
            flush.fill_(1.0)
            torch.cuda._sleep(200_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            plan.fill(n0, n1, out=out)
            b.record(st)
            fs.append((a, b))
        torch.cuda.synchronize()
        fill_ms = statistics.median(x.elapsed_time(y) for x, y in fs)
        m = prob.m
        fill_bytes = 12 * nnz + 8 * (m + 1) * 2 + 8 * m
        print(json.dumps({"N": n, "M": m, "nnz_q0": out[0].nnz, "nnz_q1": out[1].nnz, "unfold_ms": ms,
                          "nnz_per_s": nnz / (ms * 1e-3), "fill_ms": fill_ms,
                          "fill_GBps": fill_bytes / (fill_ms * 1e-3) / 1e9,
                          "output_GB": (fill_bytes) / 1e9,
                          "mem_allocated_GB": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
        plan.close()
        del out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
