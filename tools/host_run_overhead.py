"""Host-side cost of plan.run() pieces at a config (diagnostics): Python allocation / struct
building / the sun_run call / the nnz readback, and the GPU-idle gap before the graph starts."""
import os
import statistics
import sys
import time
import ctypes

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_1812_11626_b200 as sun
    from paper_1812_11626_b200 import _lib
    from workloads import config

    prob = config(int(sys.argv[1]) if len(sys.argv) > 1 else 4)
    H0 = sun.DeviceZCSR.from_host(prob.H0)
    H1 = sun.DeviceZCSR.from_host(prob.H1) if prob.H1 is not None else None
    Ls = [sun.DeviceZCSR.from_host(x) for x in prob.Ls]
    plan = sun.Plan(H0, H1, Ls, prob.gammas)
    keep = []
    for _ in range(5):
        keep.append(plan.run())
        keep = keep[-2:]
    L = sun.lib()
    st = torch.cuda.current_stream()
    rec = {k: [] for k in ("run_total", "alloc", "structs", "sun_run", "plan_nnz", "trim")}
    for it in range(40):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = plan.run()
        t1 = time.perf_counter()
        keep.append(out)
        keep = keep[-2:]
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        bufs = plan._alloc(*plan._caps)
        t3 = time.perf_counter()
        s0, s1 = plan._structs(bufs)
        t4 = time.perf_counter()
        L.sun_run(plan._plan, ctypes.addressof(s0), ctypes.addressof(s1) if s1 is not None else None,
                  bufs[2].data_ptr(), st.cuda_stream)
        t5 = time.perf_counter()
        a, b = ctypes.c_int64(), ctypes.c_int64()
        L.sun_plan_nnz(plan._plan, ctypes.addressof(a), ctypes.addressof(b))
        t6 = time.perf_counter()
        plan._trim(bufs, a.value, b.value)
        t7 = time.perf_counter()
        keep.append(bufs)
        keep = keep[-2:]
        if it >= 5:
            for k, v in zip(rec, (t1 - t0, t3 - t2, t4 - t3, t5 - t4, t6 - t5, t7 - t6)):
                rec[k].append(v)
    for k, v in rec.items():
        print(f"{k:12s} median {statistics.median(v) * 1e6:8.1f} us")


if __name__ == "__main__":
    main()
