"""Time the batched dense unfold (sun_unfold_dense) at N = 100 on one GPU.

Reports time per realisation, algorithmic bytes (A + H read, Q + K written) per realisation
and the achieved fraction of the measured HBM bandwidth; also each kernel's share of a call
(CUDA events around single-kernel runs are not available through the ABI, so the per-kernel
split comes from the ncu launch list; see profiles/)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--chunk", type=int, default=2)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    import torch

    import paper_1812_11626_b200 as sun
    from workloads import gks_ensemble_torch

    n, B = args.n, args.batch
    m = n * n - 1
    t0 = time.perf_counter()
    H, A = gks_ensemble_torch(n, B, seed=11)
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    Q = torch.empty((B, m, m), dtype=torch.float64, device="cuda")
    K = torch.empty((B, m), dtype=torch.float64, device="cuda")
    nb = sun.dense_work_bytes(n, args.chunk)
    work = torch.empty((nb + 15) // 16, dtype=torch.complex128, device="cuda")
    for _ in range(args.warmup):
        sun.unfold_dense(H, A, Q, K, work)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sun.unfold_dense(H, A, Q, K, work)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = min(ts)
    alg = B * (16 * m * m + 16 * n * n + 8 * m * m + 8 * m)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6454.6)
    out = {
        "n": n, "m": m, "batch": B, "chunk": args.chunk, "call_ms": t * 1e3, "ms_per_realisation": t * 1e3 / B,
        "realisations_per_s": B / t, "alg_bytes_per_realisation": alg // B, "alg_GBps": alg / t / 1e9,
        "frac_hbm": alg / t / 1e9 / peak, "launches": sun.lib().sun_dense_launches(n, B, 1, nb),
        "input_generation_s": gen_s, "q_finite": bool(torch.isfinite(Q).all().item()),
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
