"""Upper bound on what removing the join's per-warp size divergence could buy:
the fused C4 join (2^28 pairs, 65,536 polygons) with the C4 size mix (4..16
vertices) against databases whose polygons all have one size."""
import numpy as np
import torch

import paper_2007_15385_b200 as vp
import workloads as W

m, npoly = 1 << 28, W.C4_POLYS
dev = torch.device("cuda:0")
off, vx, vy, cx, cy, r = W.c4_polygons(vp.random_convex_polygon)
dbs = {"mix 4..16": (off, vx, vy)}
for n in (4, 8, 10, 12, 16):
    o = np.arange(npoly + 1, dtype=np.uint32) * n
    X, Y = np.empty(npoly * n), np.empty(npoly * n)
    for k in range(npoly):
        X[k * n:(k + 1) * n], Y[k * n:(k + 1) * n] = vp.random_convex_polygon(
            n, 1000 + k, float(r[k]), (float(cx[k]), float(cy[k])))
    dbs[f"all n={n}"] = (o, X, Y)
xs = torch.empty(m, dtype=torch.float32, device=dev)
ys = torch.empty(m, dtype=torch.float32, device=dev)
ids = torch.empty(m, dtype=torch.int32, device=dev)
t = lambda a: torch.from_numpy(np.asarray(a)).to(dev)
vp.fill_join_pairs(W.c4_pair_seed(), 0, xs, ys, ids, t(cx), t(cy), t(r))
words = [torch.empty((m + 31) // 32, dtype=torch.int32, device=dev) for _ in range(3)]
counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(3)]
for name, (o, X, Y) in dbs.items():
    with vp.PolygonDB.prepare(o, X, Y) as db:
        for _ in range(3):
            db.test_multi(xs, ys, ids, words=words, counts=counts)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            ev[0].record(); db.test_multi(xs, ys, ids, words=words, counts=counts); ev[1].record()
            torch.cuda.synchronize(); ts.append(ev[0].elapsed_time(ev[1]))
        print(f"{name:12s} {np.median(ts):.3f} ms", flush=True)
