"""Device time of the general-pattern (mode 3) unfold on its workloads: sun_run step and the fill
alone (CUDA events, L2 flushed), plus nnz/s and the fill's HBM fraction on algorithmic bytes.
SUNFOLD_LIB selects an experiment build.  Usage: python tools/time_general.py [names...]"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_11626_b200 as sun  # noqa: E402
from workloads import (dense_dissipator_problem, random_sparse_problem, ring_dimer_problem)  # noqa: E402

W = {
    "sparse300": lambda: random_sparse_problem(300, seed=21, P=2),
    "ring256": lambda: ring_dimer_problem(256, drive=True),
    "dense48": lambda: dense_dissipator_problem(48, seed=0),
    "dense24": lambda: dense_dissipator_problem(24, seed=0),
    "sparse1000": lambda: random_sparse_problem(1000, seed=22, P=2),
    "dense100": lambda: dense_dissipator_problem(100, seed=0),
    "ring1000": lambda: ring_dimer_problem(1000, drive=True),
}
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6454.6
names = sys.argv[1:] or ["sparse300", "ring256", "dense48"]
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for nm in names:
    prob = W[nm]()
    plan = sun.Plan(prob.H0, prob.H1, prob.Ls, prob.gammas)
    for _ in range(2):
        out = plan.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        out = plan.run()
        b.record(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    step = statistics.median([a.elapsed_time(b) for a, b in ts])
    plan.set_graphs(False)
    plan.count()
    n0, n1 = plan.nnz()
    bufs = plan.fill(n0, n1)
    fs = []
    for _ in range(10):
        flush.fill_(1.0)
        torch.cuda._sleep(200_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        plan.fill(n0, n1, out=bufs)
        b.record(st)
        fs.append((a, b))
    torch.cuda.synchronize()
    fill = statistics.median([a.elapsed_time(b) for a, b in fs])
    m = prob.m
    nnz = n0 + n1
    fb = 8 * (m + 1) + 12 * n0 + 8 * m + ((8 * (m + 1) + 12 * n1) if n1 else 0)
    print(json.dumps({"workload": nm, "N": prob.n, "nnz": nnz, "step_ms": step, "fill_ms": fill,
                      "nnz_per_s": nnz / step * 1e3, "fill_frac": fb / (fill * 1e-3) / 1e9 / peak}), flush=True)
    plan.close()
    del out, bufs
    torch.cuda.empty_cache()
