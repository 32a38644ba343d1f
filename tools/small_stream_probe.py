"""What a plain read stream reaches at C2's size (136 MB, L2 flushed): the
ceiling for a 2^24-point f32 batch, against the slab kernel."""
import torch

m = 1 << 24
x = torch.rand(2 * m, device="cuda")
flush = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
for label, fn in (("torch.sum (136 MB)", lambda: x.sum()),
                  ("torch.amax (136 MB)", lambda: x.amax())):
    ts = []
    for r in range(25):
        sink.copy_(flush.view(torch.int64).sum().view(1))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if r >= 5:
            ts.append(a.elapsed_time(b))
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"{label}: {ms * 1e3:.1f} us median, {2 * m * 4 / (ms * 1e-3) / 1e12:.2f} TB/s")
