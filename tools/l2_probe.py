"""L2 vs HBM bandwidth probe: torch copy_ of buffers of growing size, back to
back (read + write bytes / time, CUDA events)."""
import torch
for mb in [4, 8, 16, 24, 32, 48, 64, 96, 128, 512, 2048]:
    n = mb * (1 << 20) // 4
    a = torch.randn(n, device="cuda")
    b = torch.empty_like(a)
    for _ in range(3):
        b.copy_(a)
    torch.cuda.synchronize()
    reps = max(10, int(4096 / mb))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        b.copy_(a)
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    print(f"copy {mb:5d} MB (footprint {2*mb} MB): {t*1e6:9.2f} us  {2*mb*(1<<20)/t/1e9:8.0f} GB/s", flush=True)
