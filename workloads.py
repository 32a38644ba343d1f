"""Seeded synthetic workloads for the five BASELINE.json configs.

No public dataset is involved (the reference benchmarks only synthetic
regular n-gons, bench.cpp:127-134); every input here is derived from the
base seed 42 (bench.hpp:40) through mix_seed (sampling.cpp:107-112), so the
GPU path and the CPU oracle see identical polygons and points.

  C1  oracle config: random 8-angle polygon, radius 1 +- 0.2, convex hull;
      2^20 f64 points uniform in [-1.5, 1.5]^2 (vpip::sample_points)
  C2  vehicle footprint: 4.8 m x 1.9 m rectangle with 0.3 m two-facet chamfers
      (12 vertices: arc points at 0/45/90 degrees per corner), random rotation;
      2^24 f32 points in 2048 Gaussian clusters of 8192 (sigma 0.3 m), centre
      angle U[0, 2pi), centre radius U[0, 50] m
  C3  n-sweep: regular n-gons, radii jittered +-5 %, random rotation, convex
      hull; 2^28 f32 points uniform in [-1.2, 1.2]^2 ("c3x": unjittered exact n)
  C5  scaling: vpip::random_convex_polygon(32, seed, 1.0); 2^31 f32 points
      uniform in [-1.5, 1.5]^2 from the counter-based stream

Uniforms not drawn by a reference sampler are counter-based:
U(seed, j) = top-53-bits(mix_seed(seed, j)) * 2^-53 (sampling.cpp:31-33).
"""
from __future__ import annotations

import math

import numpy as np

BASE_SEED = 42
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix_seed_np(seed: int, salt) -> np.ndarray:
    """Vectorised splitmix64 finaliser (sampling.cpp:107-112) over uint64 salts."""
    with np.errstate(over="ignore"):
        s = np.asarray(salt, dtype=np.uint64)
        z = np.uint64(seed) + np.uint64(0x9E3779B97F4A7C15) * (s + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def unit_np(seed: int, salt) -> np.ndarray:
    return (mix_seed_np(seed, salt) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def config_seed(config: int) -> int:
    return int(mix_seed_np(BASE_SEED, config))


def convex_hull(px, py):
    """Strict convex hull (Andrew's monotone chain, collinear points dropped), CCW,
    starting from the lowest-x (then lowest-y) vertex."""
    pts = sorted(set(zip(map(float, px), map(float, py))))
    if len(pts) < 3:
        return np.array([p[0] for p in pts]), np.array([p[1] for p in pts])

    def cross(o, a, b):
        return (a[0] - o[0]) * (b[1] - o[1]) - (a[1] - o[1]) * (b[0] - o[0])

    lower, upper = [], []
    for p in pts:
        while len(lower) >= 2 and cross(lower[-2], lower[-1], p) <= 0:
            lower.pop()
        lower.append(p)
    for p in reversed(pts):
        while len(upper) >= 2 and cross(upper[-2], upper[-1], p) <= 0:
            upper.pop()
        upper.append(p)
    hull = lower[:-1] + upper[:-1]
    return np.array([p[0] for p in hull]), np.array([p[1] for p in hull])


# ---------------------------------------------------------------- C1
def c1_polygon(seed: int | None = None):
    """8 sorted uniform angles, radius 1 +- 0.2 (uniform), convex hull, origin-centred."""
    seed = config_seed(1) if seed is None else seed
    ang = np.sort(2.0 * math.pi * unit_np(seed, np.arange(8)))
    rad = 1.0 + 0.2 * (2.0 * unit_np(seed, 8 + np.arange(8)) - 1.0)
    return convex_hull(rad * np.cos(ang), rad * np.sin(ang))


C1_POINTS = 1 << 20
C1_BOX = (-1.5, -1.5, 1.5, 1.5)


def c1_points(sample_points, count: int = C1_POINTS):
    """`sample_points` = vpip::sample_points semantics (product or oracle sampler)."""
    return sample_points(count, C1_BOX, mix_seed_np(config_seed(1), 100).item())


# ---------------------------------------------------------------- C2
C2_CLUSTERS, C2_PER_CLUSTER, C2_SIGMA, C2_RMAX = 2048, 8192, 0.3, 50.0


def c2_polygon(seed: int | None = None):
    seed = config_seed(2) if seed is None else seed
    a, b, r = 2.4, 0.95, 0.3
    corners = [(a - r, b - r, 0.0), (-(a - r), b - r, 90.0), (-(a - r), -(b - r), 180.0),
               ((a - r), -(b - r), 270.0)]
    vx, vy = [], []
    for cx, cy, start in corners:
        for t in (0.0, 45.0, 90.0):
            th = math.radians(start + t)
            vx.append(cx + r * math.cos(th))
            vy.append(cy + r * math.sin(th))
    phi = 2.0 * math.pi * unit_np(seed, 0).item()
    c, s = math.cos(phi), math.sin(phi)
    vx, vy = np.array(vx), np.array(vy)
    return c * vx - s * vy, s * vx + c * vy


def c2_points(seed: int | None = None, clusters: int = C2_CLUSTERS):
    """Gaussian clusters (Box-Muller on counter-based uniforms), float32."""
    seed = config_seed(2) if seed is None else seed
    k = np.arange(clusters, dtype=np.uint64)
    cang = 2.0 * math.pi * unit_np(seed, 1000 + 2 * k)
    crad = C2_RMAX * unit_np(seed, 1001 + 2 * k)
    cx = np.repeat(crad * np.cos(cang), C2_PER_CLUSTER)
    cy = np.repeat(crad * np.sin(cang), C2_PER_CLUSTER)
    j = np.arange(clusters * C2_PER_CLUSTER, dtype=np.uint64)
    pseed = int(mix_seed_np(seed, 7))
    u1 = 1.0 - unit_np(pseed, 2 * j)  # (0, 1]
    u2 = unit_np(pseed, 2 * j + 1)
    rr = C2_SIGMA * np.sqrt(-2.0 * np.log(u1))
    return ((cx + rr * np.cos(2 * math.pi * u2)).astype(np.float32),
            (cy + rr * np.sin(2 * math.pi * u2)).astype(np.float32))


# ---------------------------------------------------------------- C3
C3_NS = (3, 4, 8, 16, 64, 256, 1024)
C3_POINTS = 1 << 28
C3_BOX = (-1.2, -1.2, 1.2, 1.2)


def c3_polygon(n: int, jitter: float = 0.05, seed: int | None = None):
    """Regular n-gon, radii jittered +-jitter, random rotation, convex hull."""
    seed = config_seed(3) if seed is None else seed
    s = int(mix_seed_np(seed, n))
    rot = 2.0 * math.pi * unit_np(s, 0).item()
    k = np.arange(n)
    rad = 1.0 + jitter * (2.0 * unit_np(s, 1 + k) - 1.0)
    ang = rot + 2.0 * math.pi * k / n
    return convex_hull(rad * np.cos(ang), rad * np.sin(ang))


def c3_named(name: str):
    """Polygon of a bench workload name: "c3:<n>" is the literal C3 config (jittered
    hull, so n_eff < n for large n); "c3x:<n>" is the unjittered exact-n
    supplement SURVEY §8d recommends (regular n-gon, random rotation, all n
    vertices strictly convex up to n = 1024) that reaches the compute-bound
    regime. Both use the C3 point stream of that n."""
    kind, _, n = name.partition(":")
    n = int(n) if n else 8
    return n, c3_polygon(n, jitter=0.0 if kind == "c3x" else 0.05)


# ---------------------------------------------------------------- C4
C4_POLYS = 65536
C4_PAIRS = 1 << 28


def c4_polygons(random_convex_polygon, npoly: int = C4_POLYS, seed: int | None = None):
    """CSR table of `npoly` vpip::random_convex_polygon(n_i, seed_i, r_i, c_i):
    n_i uniform in {4..16}, c_i uniform in [0, 1000]^2, r_i uniform in [0.5, 5].
    Returns offsets (u32, npoly+1), vx, vy, and per-polygon cx, cy, r."""
    s = config_seed(4) if seed is None else seed
    i = np.arange(npoly, dtype=np.uint64)
    n = 4 + np.minimum((unit_np(s, 4 * i) * 13).astype(np.int64), 12)
    cx = 1000.0 * unit_np(s, 4 * i + 1)
    cy = 1000.0 * unit_np(s, 4 * i + 2)
    r = 0.5 + 4.5 * unit_np(s, 4 * i + 3)
    seeds = mix_seed_np(int(mix_seed_np(s, 103)), i)
    offsets = np.zeros(npoly + 1, dtype=np.uint32)
    offsets[1:] = np.cumsum(n)
    vx = np.empty(int(offsets[-1]))
    vy = np.empty(int(offsets[-1]))
    for k in range(npoly):
        a, b = int(offsets[k]), int(offsets[k + 1])
        vx[a:b], vy[a:b] = random_convex_polygon(int(n[k]), int(seeds[k]), float(r[k]),
                                                 (float(cx[k]), float(cy[k])))
    return offsets, vx, vy, cx, cy, r


def c4_pair_seed() -> int:
    return int(mix_seed_np(config_seed(4), 102))


# ---------------------------------------------------------------- C5
C5_POINTS = 1 << 31
C5_BOX = (-1.5, -1.5, 1.5, 1.5)
C5_EDGES = 32


def c5_polygon(random_convex_polygon, seed: int | None = None):
    """`random_convex_polygon` = vpip::random_convex_polygon semantics."""
    seed = config_seed(5) if seed is None else seed
    return random_convex_polygon(C5_EDGES, seed, 1.0)


def c5_point_seed() -> int:
    return int(mix_seed_np(config_seed(5), 101))


def shard(m: int, rank: int, world: int, align: int = 1024):
    """Contiguous, `align`-aligned point range of one rank (masks concatenate)."""
    from paper_2007_15385_b200.multi import shard as _shard
    return _shard(m, rank, world, align)
