import time, sys, torch
sys.path.insert(0, '.')
import paper_2007_15385_b200 as vp
import workloads as W
m = 1 << 31
hx = torch.empty(m, dtype=torch.float32, pin_memory=True)
hy = torch.empty(m, dtype=torch.float32, pin_memory=True)
hx.uniform_(-1.5, 1.5); hy.uniform_(-1.5, 1.5)
dx = torch.empty(m, dtype=torch.float32, device='cuda'); dy = torch.empty_like(dx)
for r in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    dx.copy_(hx, non_blocking=True); dy.copy_(hy, non_blocking=True); torch.cuda.synchronize()
    print("pure h2d 17.2GB: %.1f ms  %.1f GB/s" % ((time.perf_counter()-t)*1e3, 2*4*m/(time.perf_counter()-t)/1e9))
del dx, dy
vx, vy = W.c5_polygon(vp.random_convex_polygon)
p = vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL, device=0)
hw = [torch.empty((m + 31) // 32, dtype=torch.int32, pin_memory=True) for _ in range(3)]
for label, words in (("multi+words", hw), ("multi no words", None)):
    for r in range(3):
        t = time.perf_counter()
        p.test_host_multi(hx, hy, (0, 1, 2), words=words, counts_only=words is None)
        dt = time.perf_counter() - t
        print("%s: %.1f ms  -> %.3e tests/s  (%.1f GB/s H2D)" % (label, dt*1e3, 3*m/dt, 8*m/dt/1e9))
