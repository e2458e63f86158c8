"""Device timeline of a few unfold steps (torch.profiler / CUPTI): per-kernel start offsets and
durations inside one plan.run() step, plus the host-side duration of the step.  Diagnostics only."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_1812_11626_b200 as sun
    from workloads import config

    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    prob = config(cfg)
    H0 = sun.DeviceZCSR.from_host(prob.H0)
    H1 = sun.DeviceZCSR.from_host(prob.H1) if prob.H1 is not None else None
    Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
    plan = sun.Plan(H0, H1, Ls, prob.gammas)
    for _ in range(5):
        out = plan.run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            torch.cuda.synchronize()
            with torch.profiler.record_function("step"):
                out = plan.run()
            torch.cuda.synchronize()
    kern = sorted([e for e in prof.events() if e.device_type.name == "CUDA" and e.name != "step"],
                  key=lambda e: e.time_range.start)
    # the last step's kernels: after the last gap > 200 us between consecutive kernels
    start = 0
    for i in range(1, len(kern)):
        if kern[i].time_range.start - max(k.time_range.end for k in kern[:i]) > 200:
            start = i
    last = kern[start:]
    t0 = last[0].time_range.start
    t1 = max(k.time_range.end for k in last)
    print(f"last step: device span {t1 - t0:.1f} us ({len(last)} device ops)")
    for k in last:
        print(f"  +{k.time_range.start - t0:8.1f} us  dur {k.time_range.end - k.time_range.start:8.1f} us  "
              f"{k.name[:70]}")
    print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))


if __name__ == "__main__":
    main()
