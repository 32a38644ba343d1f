#!/usr/bin/env python3
"""run_benchmark (proj/src/bench.cpp:115-222) on the B200 drop-in, with records
in the reference CSV schema (bench.cpp:224-234) -- SURVEY.md §8(f)4.

Methodology mirrors the reference's:
- one regular n-gon (r = 1) per edge count;
- one pre-sampled batch per n over the polygon's bounding box scaled 2x, from
  vpip::sample_points with seed mix_seed(seed, n);
- conversion timed once (Voronoi, `phase=convert`: vpipg_prepare, i.e.
  validation + the device to_voronoi, synchronous);
- one discarded warm-up per (engine, n);
- `repetitions` rounds in a seeded shuffled order, each record timing exactly
  the drop-in batch call (vpipg_test_host: host f64 batch in, byte mask out,
  the path behind vpip::*_contains_batch).

    python tools/gpu_run_benchmark.py [--batch 1000000] [--reps 10] [--out gpu_bench.csv]
"""
from __future__ import annotations

import argparse
import random
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2007_15385_b200 as vp  # noqa: E402

ENGINES = ("voronoi", "sign_of_offset", "ray_crossing")
HEADER = "engine,n_edges,batch_size,repetition,phase,wall_time_ns,throughput_pts_per_s"


def box_scaled(vx, vy, factor=2.0):
    """Box::scaled of bounding_box (geometry.hpp:64-69)."""
    x0, x1, y0, y1 = vx.min(), vx.max(), vy.min(), vy.max()
    cx, cy = 0.5 * (x0 + x1), 0.5 * (y0 + y1)
    hw, hh = 0.5 * factor * (x1 - x0), 0.5 * factor * (y1 - y0)
    return (cx - hw, cy - hh, cx + hw, cy + hh)


def run_benchmark(edge_counts=range(3, 16), batch=1_000_000, reps=10, seed=42, device=0):
    work = []
    for n in edge_counts:
        vx, vy = vp.regular_polygon(n, 1.0)
        xs, ys = vp.sample_points(batch, box_scaled(vx, vy), vp.mix_seed(seed, n))
        work.append((n, vx, vy, xs, ys))
    records, handles = [], {}
    for e, name in enumerate(ENGINES):
        for n, vx, vy, xs, ys in work:
            kind = (vp.KIND_VORONOI, vp.KIND_OFFSET, vp.KIND_CROSSING)[e]
            t0 = time.perf_counter_ns()
            h = vp.PreparedPolygon.prepare(vx, vy, kind, device=device)
            t1 = time.perf_counter_ns()
            if e == 0:
                records.append((name, n, 0, 0, "convert", max(t1 - t0, 1), 0.0))
            handles[(e, n)] = h
            h.test_host(e, xs, ys, words=False, bytes_=True)  # discarded warm-up
    queries = {}
    order = [(e, i) for e in range(3) for i in range(len(work))]
    for rep in range(reps):
        random.Random(vp.mix_seed(seed, 0x0BEF0000 + rep)).shuffle(order)
        for e, i in order:
            n, vx, vy, xs, ys = work[i]
            t0 = time.perf_counter_ns()
            handles[(e, n)].test_host(e, xs, ys, words=False, bytes_=True)
            ns = max(time.perf_counter_ns() - t0, 1)
            queries.setdefault((e, i), []).append((ENGINES[e], n, batch, rep, "query", ns,
                                                   batch / (ns * 1e-9)))
    out = [r for r in records]
    canon = []
    for e in range(3):
        for i, (n, *_rest) in enumerate(work):
            if e == 0:
                canon += [r for r in records if r[1] == n]
            canon += queries[(e, i)]
    for h in handles.values():
        h.close()
    return canon


def to_csv(records) -> str:
    lines = [HEADER]
    for eng, n, b, rep, phase, ns, tp in records:
        lines.append(f"{eng},{n},{b},{rep},{phase},{ns},{tp:.17g}")
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="gpu_bench.csv")
    a = ap.parse_args()
    csv = to_csv(run_benchmark(batch=a.batch, reps=a.reps))
    Path(a.out).write_text(csv)
    print(f"wrote {a.out}")


if __name__ == "__main__":
    main()
