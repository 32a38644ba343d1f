"""Host-buffer drop-in throughput: pageable numpy vs pinned torch buffers (vpipg_test_host)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2007_15385_b200 as vp  # noqa: E402

vx, vy = vp.regular_polygon(8, 1.0)
with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
    for m in (1 << 20, 1 << 24, 1 << 26):
        xs, ys = vp.sample_points(m, (-2, -2, 2, 2), 5)
        px = torch.from_numpy(xs).pin_memory().numpy()
        py = torch.from_numpy(ys).pin_memory().numpy()
        for label, (a, b) in (("pageable", (xs, ys)), ("pinned", (px, py))):
            for out in ("bytes", "words"):
                ts = []
                for r in range(4):
                    t0 = time.perf_counter()
                    p.test_host(0, a, b, words=(out == "words"), bytes_=(out == "bytes"))
                    ts.append(time.perf_counter() - t0)
                t = min(ts[1:])
                print(f"m={m:>9d} {label:8s} {out:5s} {t * 1e3:8.2f} ms  {m / t:.3e} pts/s  "
                      f"{16 * m / t / 1e9:.1f} GB/s in")
