"""Host-side cost of one vpipg_test call (small batch, device buffers)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2007_15385_b200 as vp  # noqa: E402

vx, vy = vp.regular_polygon(8, 1.0)
m = 4096
xs = torch.rand(m, device="cuda") * 2 - 1
ys = torch.rand(m, device="cuda") * 2 - 1
w = torch.zeros(m // 32, dtype=torch.int32, device="cuda")
with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
    for e in range(3):
        for _ in range(10):
            p.test(e, xs, ys, words=w)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(1000):
            p.test(e, xs, ys, words=w)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"engine {e}: {(t1 - t0) * 1e3:.1f} us host per call, {(t2 - t0) * 1e3:.1f} us per call incl. GPU")
