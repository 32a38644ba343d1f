"""Generate tests/golden/reference_fixtures.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference; oracle/Makefile compiles the
reference sources into oracle/_ref/libvpip_ref.so):

    python tests/golden/make_golden.py

Every output value comes from the reference library itself (vpip::sample_points,
regular_polygon, random_convex_polygon, validate_polygon, to_voronoi and the
three *_contains_batch engines). The fixtures pin both the C restatement
(tests/test_oracle_golden.py, CPU) and the GPU engine (tests/test_gpu_parity.py)
without /root/reference at run time.
"""
from __future__ import annotations

import hashlib
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "reference_fixtures.npz"


def main() -> None:
    oracle.build(ref=True)
    R = oracle.Reference()
    L = R.L
    fx: dict[str, np.ndarray] = {}
    ms = lambda s, t: int(L.vr_mix_seed(s, t))

    # --- sampling (sampling.cpp) ---
    seeds = [0, 1, 42, 4242, 2**63 + 5, 2**64 - 1]
    fx["mix_seed_in"] = np.array([(s, t) for s in seeds for t in (0, 1, 7, 2**40)], np.uint64)
    fx["mix_seed_out"] = np.array([ms(int(s), int(t)) for s, t in fx["mix_seed_in"]], np.uint64)
    xs, ys = R.sample_points(1000, (-1, -1, 2, 2), 4242)
    fx["sample_xs"], fx["sample_ys"] = xs, ys
    for n in range(3, 17):
        fx[f"regular_{n}"] = np.stack(R.regular_polygon(n, 1.0))
    rcp = [(n, s) for n in (3, 4, 7, 8, 12, 16, 32) for s in (1, 99, ms(1001, n))]
    fx["rcp_params"] = np.array(rcp, np.uint64)
    for i, (n, s) in enumerate(rcp):
        fx[f"rcp_{i}"] = np.stack(R.random_convex_polygon(n, s, 1.0))

    # --- validation error codes (geometry.cpp:53-98) ---
    bad = {
        "too_few": ([0, 1], [0, 0]),
        "nonfinite": ([0, 1, np.inf], [0, 0, 1]),
        "degenerate": ([0, 1, 1, 0], [0, 0, 0, 0]),
        "collinear": ([0, 1, 2, 1], [0, 0, 0, 1]),
        "reflex": ([0, 4, 4, 2, 0], [0, 0, 4, 1, 4]),
        "pentagram": ([math.cos(2 * math.pi * (2 * k) / 5) for k in range(5)],
                      [math.sin(2 * math.pi * (2 * k) / 5) for k in range(5)]),
        "clockwise_square": ([0, 0, 1, 1], [0, 1, 1, 0]),
    }
    for name, (vx, vy) in bad.items():
        rc, ox, oy, rev = R.validate(vx, vy)
        fx[f"val_{name}_in"] = np.array([vx, vy], np.float64)
        fx[f"val_{name}_code"] = np.array(rc)
        fx[f"val_{name}_out"] = np.array([ox, oy])
        fx[f"val_{name}_rev"] = np.array(rev)

    # --- conversion (voronoi.cpp:60-71) ---
    conv = [("unit_square", [0, 1, 1, 0], [0, 0, 1, 1]), ("triangle", [0, 1, 0], [0, 0, 1])]
    conv.append(("pentagon",) + tuple(R.regular_polygon(5, 1.0)))
    for i in range(50):  # test_voronoi.cpp:33-39 make_test_polygon
        n = 3 + ms(11, i) % 13
        rad = 0.5 + 2.5 * (ms(12, i) % 100) / 100.0
        c = (float(ms(13, i) % 9) - 4.0, float(ms(14, i) % 9) - 4.0)
        conv.append((f"tv{i}",) + tuple(R.random_convex_polygon(n, ms(15, i), rad, c)))
    conv.append(("c1",) + tuple(W.c1_polygon()))
    conv.append(("c2",) + tuple(W.c2_polygon()))
    conv.append(("c5",) + tuple(R.random_convex_polygon(32, W.config_seed(5), 1.0)))
    for n in W.C3_NS:
        conv.append((f"c3_{n}",) + tuple(W.c3_polygon(n)))
    fx["conv_names"] = np.array([c[0] for c in conv])
    for name, vx, vy in conv:
        rc, inner, outer = R.to_voronoi(vx, vy)
        assert rc == 0, (name, rc)
        fx[f"conv_{name}_v"] = np.array([vx, vy], np.float64)
        fx[f"conv_{name}_inner"] = inner
        fx[f"conv_{name}_outer"] = outer

    # --- engine masks (engines.cpp), three engines per case ---
    cases = []

    def edge_probes(vx, vy, rng_seed):
        """Vertices, midpoints and points a hair off every edge line."""
        vx, vy = np.asarray(vx, float), np.asarray(vy, float)
        n = vx.size
        px, py = list(vx), list(vy)
        g = np.random.default_rng(rng_seed)
        for k in range(n):
            k1 = (k + 1) % n
            for t in (0.5, 0.25, g.random()):
                x = vx[k] + t * (vx[k1] - vx[k])
                y = vy[k] + t * (vy[k1] - vy[k])
                nx, ny = vy[k1] - vy[k], -(vx[k1] - vx[k])
                nn = math.hypot(nx, ny)
                for off in (0.0, 1e-12, -1e-12, 1e-7, -1e-7):
                    px.append(x + off * nx / nn)
                    py.append(y + off * ny / nn)
        return np.array(px), np.array(py)

    def add_case(name, vx, vy, xs, ys, f32=False):
        vx, vy = np.asarray(vx, np.float64), np.asarray(vy, np.float64)
        xs, ys = np.asarray(xs, np.float64), np.asarray(ys, np.float64)
        if f32:  # both sides see the same f32-rounded polygon and points
            vx, vy = vx.astype(np.float32).astype(np.float64), vy.astype(np.float32).astype(np.float64)
            xs, ys = xs.astype(np.float32).astype(np.float64), ys.astype(np.float32).astype(np.float64)
        (mv, mo, mr), _ = R.masks(vx, vy, xs, ys)
        pairs, dis, ok = R.run_validation(vx, vy, xs, ys, band=1e-9)  # bench.cpp:279-308
        fx[f"case_{name}_validation"] = np.array(pairs + [dis, int(ok)], np.int64)
        cases.append(name)
        p = f"case_{name}_"
        fx[p + "v"] = np.array([vx, vy])
        fx[p + "pts"] = np.array([xs, ys], np.float32 if f32 else np.float64)
        fx[p + "masks"] = np.packbits(np.array([mv, mo, mr]), axis=1, bitorder="little")
        fx[p + "f32"] = np.array(f32)

    sq = ([0, 1, 1, 0], [0, 0, 1, 1])
    add_case("unit_square_known", *sq, [0.5, 2, 1, 0.5, 2, 0, 1, 1, 0, 0.5, 1, 0.5],
             [0.5, 2, 0.5, 0.5, 0.5, 0, 0, 1, 1, 0, 0.5, 1])
    xs, ys = R.sample_points(10000, (-1, -1, 2, 2), 4242)  # test_engines.cpp:139-144
    add_case("unit_square_4242", *sq, xs, ys)
    for i in range(12):  # test_engines.cpp:32-38 make_test_polygon, :146-160
        n = 3 + ms(21, i) % 13
        rad = 0.5 + 2.0 * (ms(22, i) % 100) / 100.0
        c = (float(ms(23, i) % 7) - 3.0, float(ms(24, i) % 7) - 3.0)
        vx, vy = R.random_convex_polygon(n, ms(25, i), rad, c)
        bx = (vx.min(), vy.min(), vx.max(), vy.max())
        cx, cy, hw, hh = (bx[0] + bx[2]) / 2, (bx[1] + bx[3]) / 2, bx[2] - bx[0], bx[3] - bx[1]
        xs, ys = R.sample_points(2000, (cx - hw, cy - hh, cx + hw, cy + hh), ms(32, i))
        ex, ey = edge_probes(vx, vy, i)
        add_case(f"te{i}", vx, vy, np.concatenate([xs, ex]), np.concatenate([ys, ey]))
    for n in (3, 8, 15):  # acceptance.cpp:98-116
        for which, (vx, vy) in enumerate([R.regular_polygon(n, 1.0),
                                          R.random_convex_polygon(n, ms(1001, n), 1.0)]):
            xs, ys = R.sample_points(2000, (-2, -2, 2, 2), ms(2001, 2 * n + which))
            add_case(f"acc_{n}_{which}", vx, vy, xs, ys)
    c1x, c1y = W.c1_polygon()
    xs, ys = R.sample_points(4096, W.C1_BOX, 12345)
    ex, ey = edge_probes(c1x, c1y, 99)
    add_case("c1_sample", c1x, c1y, np.concatenate([xs, ex]), np.concatenate([ys, ey]))
    # clockwise input: validation reverses it, crossing keeps the raw order
    add_case("c1_clockwise", c1x[::-1], c1y[::-1], xs[:1024], ys[:1024])
    # f32 configs (C2, C3, C5): f32-rounded polygon + points
    c2x, c2y = W.c2_polygon()
    px, py = W.c2_points(clusters=2)
    add_case("c2_f32", c2x, c2y, px[::4][:4096], py[::4][:4096], f32=True)
    for n in W.C3_NS:
        vx, vy = W.c3_polygon(n)
        xs, ys = R.sample_points(2048, W.C3_BOX, ms(3000, n))
        add_case(f"c3_{n}_f32", vx, vy, xs, ys, f32=True)
    c5x, c5y = R.random_convex_polygon(32, W.config_seed(5), 1.0)
    o = oracle.Oracle()
    xs, ys = o.counter_points_f32(W.c5_point_seed(), 0, 4096, W.C5_BOX)
    add_case("c5_f32", c5x, c5y, xs, ys, f32=True)
    fx["case_names"] = np.array(cases)

    # concave arrow (test_engines.cpp:73-81): crossing only
    ax, ay = np.array([0, 4, 4, 2, 0], float), np.array([0, 0, 4, 1, 4], float)
    code = np.zeros(1, np.int32)
    import ctypes as C
    p = L.vr_poly_new(ax.ctypes.data_as(oracle._D), ay.ctypes.data_as(oracle._D), 5, 0,
                      C.cast(code.ctypes.data, C.POINTER(C.c_int)))
    probes = [(2, 2), (1, 1), (3, 1), (-1, 1), (2, 1), (4, 2), (0, 0)]
    fx["arrow_v"] = np.array([ax, ay])
    fx["arrow_pts"] = np.array(probes, float).T
    fx["arrow_inside"] = np.array([L.vr_scalar(p, 2, x, y) for x, y in probes], np.uint8)
    fx["arrow_count"] = np.array([L.vr_scalar(p, 3, x, y) for x, y in probes], np.int32)
    L.vr_poly_free(p)

    # --- non-finite and extreme query points (outside the reference's I/O
    # contract, parse_points_csv rejects NaN, but the batch kernels still give
    # a defined IEEE answer that the f64 engines must repeat) ---
    inf, nan = np.inf, np.nan
    special = [(inf, 0), (-inf, 0), (0, inf), (0, -inf), (inf, inf), (-inf, -inf), (inf, -inf),
               (nan, 0), (0, nan), (nan, nan), (inf, nan), (nan, -inf), (1e300, 1e300),
               (-1e308, 5), (5, 1.7e308), (1e-320, 0), (-0.0, -0.0), (0.1, 0.1), (3, 3)]
    sx, sy = np.array(special, float).T
    for name, (vx, vy) in (("c1", (c1x, c1y)), ("square", sq)):
        vx, vy = np.asarray(vx, float), np.asarray(vy, float)
        (mv, mo, mr), _ = R.masks(vx, vy, sx, sy)
        fx[f"nonfinite_{name}_v"] = np.array([vx, vy])
        fx[f"nonfinite_{name}_pts"] = np.array([sx, sy])
        fx[f"nonfinite_{name}_masks"] = np.array([mv, mo, mr], np.uint8)

    # --- C1 at full size: counts + SHA-256 of the packed masks ---
    xs, ys = R.sample_points(W.C1_POINTS, W.C1_BOX, W.mix_seed_np(W.config_seed(1), 100).item())
    (mv, mo, mr), _ = R.masks(c1x, c1y, xs, ys, threads=8)
    fx["c1_full_counts"] = np.array([mv.sum(), mo.sum(), mr.sum()], np.int64)
    fx["c1_full_sha256"] = np.array([hashlib.sha256(np.packbits(m, bitorder="little").tobytes()).hexdigest()
                                     for m in (mv, mo, mr)])
    fx["c1_first_xy"] = np.array([xs[:8], ys[:8]])

    np.savez_compressed(OUT, **fx)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(cases)} mask cases)")


if __name__ == "__main__":
    main()
