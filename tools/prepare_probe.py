"""Latency of vpipg_prepare (validation + device to_voronoi + tables) for one polygon."""
import sys
import time

sys.path.insert(0, ".")
import paper_2007_15385_b200 as vp  # noqa: E402

for n in (8, 32, 1024):
    vx, vy = vp.regular_polygon(n, 1.0)
    ts = []
    for r in range(50):
        t0 = time.perf_counter()
        p = vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL)
        ts.append(time.perf_counter() - t0)
        p.close()
    ts.sort()
    print(f"n={n}: first {ts[-1] * 1e3:.2f} ms, median {ts[len(ts) // 2] * 1e6:.0f} us, min {ts[0] * 1e6:.0f} us")
