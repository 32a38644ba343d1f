"""H2D / D2H bandwidth from pinned memory on this box (context for the e2e number)."""
import time
import torch

for mb in (256, 1024, 4096):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    for direction in ("h2d", "d2h"):
        src, dst = (h, d) if direction == "h2d" else (d, h)
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print(f"{direction} {mb} MiB: {n / dt / 1e9:.1f} GB/s")
