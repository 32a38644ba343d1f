"""Throughput of the exact f64 kernels (the vpip:: drop-in path) on device-resident points."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2007_15385_b200 as vp
import workloads as W

m = 1 << 27
xs = torch.empty(m, dtype=torch.float64, device="cuda")
ys = torch.empty_like(xs)
vp.fill_uniform_points(W.c5_point_seed(), 0, xs, ys, W.C5_BOX)
for n in (8, 32):
    vx, vy = vp.random_convex_polygon(n, 7, 1.0)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        w = torch.empty((m + 31) // 32, dtype=torch.int32, device="cuda")
        for e in range(3):
            p.test(e, xs, ys, words=w)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(3):
                p.test(e, xs, ys, words=w)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 3
            print(f"n={n} engine={e} {ms:.2f} ms  {m / ms / 1e6:.3e} pts/s  {m * n / ms / 1e6:.3e} pe/s  {m * 16 / ms / 1e6:.0f} GB/s")
