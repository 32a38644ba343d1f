"""C5-size step: three separate engine kernels vs the fused one-read pass."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2007_15385_b200 as vp  # noqa: E402
import workloads as W  # noqa: E402

for label, m in (("C5 2^31", 1 << 31), ("C3-like 2^28", 1 << 28)):
    n = 32 if m == 1 << 31 else 3
    vx, vy = (W.c5_polygon(vp.random_convex_polygon) if n == 32 else vp.regular_polygon(3, 1.0))
    xs = torch.empty(m, dtype=torch.float32, device="cuda")
    ys = torch.empty_like(xs)
    vp.fill_uniform_points(W.c5_point_seed(), 0, xs, ys, (-1.5, -1.5, 1.5, 1.5))
    ws = [torch.empty(m // 32, dtype=torch.int32, device="cuda") for _ in range(3)]
    cs = [torch.zeros(1, dtype=torch.int64, device="cuda") for _ in range(3)]
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        def sep():
            for e in range(3):
                p.test(e, xs, ys, words=ws[e], count=cs[e])
        def fused():
            p.test_multi(xs, ys, (0, 1, 2), words=ws, counts=cs)
        for name, fn in (("separate", sep), ("fused", fused), ("separate", sep), ("fused", fused)):
            fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(5):
                fn()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 5
            print(f"{label} n={n} {name}: {ms:.3f} ms/step  {3 * m / ms / 1e9:.3e} tests/s")
    del xs, ys, ws
    torch.cuda.empty_cache()
