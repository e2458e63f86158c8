"""sun_run step with and without phase timing (event-record nodes), and the in-pipeline count /
fill phase times (diagnostics)."""
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
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream()
    for rep in range(2):
        for timing in (False, True):
            plan.set_timing(timing)
            keep, ts, ph = [], [], []
            for i in range(60):
                flush.fill_(1.0)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                out = plan.run()
                b.record(st)
                keep.append(out)
                keep = keep[-2:]
                if i >= 10:
                    ts.append((a, b))
                    if timing:
                        ph.append(plan.phase_ms())
            torch.cuda.synchronize()
            step = statistics.mean(a.elapsed_time(b) for a, b in ts) * 1e3
            msg = f"timing={timing} step {step:.1f} us"
            if ph:
                msg += f" count {statistics.mean(c for c, f in ph) * 1e3:.1f} us fill {statistics.mean(f for c, f in ph) * 1e3:.1f} us"
            print(msg)


if __name__ == "__main__":
    main()
