"""Write-only and copy bandwidth on this GPU (CUDA events): the ceiling for an output-bound kernel."""
import torch

torch.cuda.synchronize()
for mb in (64, 128, 257, 1024, 4096):
    n = mb * (1 << 20) // 8
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name, fn, nbytes in (("fill_", lambda: x.fill_(1.0), n * 8), ("zero_", lambda: x.zero_(), n * 8),
                             ("copy_", lambda: y.copy_(x), 2 * n * 8)):
        ts = []
        for it in range(12):
            flush.fill_(it & 255)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = sorted(ts[2:])[len(ts[2:]) // 2]
        print(f"{mb:5d} MB {name}: {t * 1e3:8.1f} us  {nbytes / t / 1e6:7.1f} GB/s", flush=True)
