"""CPU legs of bench.py: the reference's own CPU implementation on the full
workload, and the parity block of the bench line.

MEASUREMENT / TEST INFRASTRUCTURE, imported only by bench.py (its
`cpu_baseline` leg, its `--impl reference` arm and its `parity` block), tests/
and __graft_entry__.smoke() as the checker. It runs
the unmodified reference library (oracle/_ref, built from /root/reference by
oracle/Makefile; the oracle port when that library is absent) and the C
oracle's edge_line_distance, never the product kernels.

Workload handling follows SURVEY.md 8(d): f32 configs are rounded to f32 and
widened exactly to f64 for the reference (it has no f32 path); C5's 2^31
points run in PointBatch chunks of 2^26 points (32 GiB of f64 in all), the
batch calls timed as run_benchmark times them (bench.cpp:196-199) and
count_inside (engines.cpp:215-217) timed as its own step; the C4 join runs as
one reference batch call per polygon over its id-grouped pairs, and the
per-pair scalar loop (engines.cpp:235-241, :304-318, :331-350) beside it.
"""
from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np

import workloads as W

CHUNK = 1 << 26          # points per reference PointBatch (1 GiB of f64)
EPS32, EPS64 = 1e-5, 1e-9  # north_star band: relative 1e-5 (f32), 1e-9 (f64)
NAMES = ("voronoi", "sign_of_offset", "ray_crossing")


def cores() -> int:
    return os.cpu_count() or 1


def host_points_f32(seed: int, m: int, box, threads: int | None = None):
    """The counter-based f32 point stream (fill.cu's, bit for bit) generated on
    the host by the C oracle, in parallel slices."""
    import oracle
    orc = oracle.Oracle()
    xs, ys = np.empty(m, np.float32), np.empty(m, np.float32)
    step = 1 << 24

    def one(lo):
        hi = min(m, lo + step)
        a, b = orc.counter_points_f32(seed, lo, hi - lo, box)
        xs[lo:hi], ys[lo:hi] = a, b

    with cf.ThreadPoolExecutor(max_workers=threads or cores()) as ex:
        list(ex.map(one, range(0, m, step)))
    return xs, ys


def reference_polygon(name: str):
    """The workload's polygon exactly as the GPU arm builds it (f64 vertices)."""
    import oracle
    orc = oracle.Oracle()
    if name == "c5":
        return W.c5_polygon(orc.random_convex_polygon)
    if name.startswith("c3"):
        return W.c3_named(name)[1]
    if name == "c2":
        return W.c2_polygon()
    return W.c1_polygon()


def host_workload(name: str, m: int | None = None):
    """Polygon + the workload's f32 points on the host (C5 / C3 / C2)."""
    vx, vy = reference_polygon(name)
    if name == "c5":
        xs, ys = host_points_f32(W.c5_point_seed(), m or W.C5_POINTS, W.C5_BOX)
    elif name.startswith("c3"):
        n = W.c3_named(name)[0]
        xs, ys = host_points_f32(int(W.mix_seed_np(W.config_seed(3), 200 + n)), m or W.C3_POINTS,
                                 W.C3_BOX)
    elif name == "c2":
        xs, ys = W.c2_points()
        if m:
            xs, ys = xs[:m], ys[:m]
    else:
        raise ValueError(name)
    return vx, vy, np.ascontiguousarray(xs, np.float32), np.ascontiguousarray(ys, np.float32)


class RefRun:
    """One workload resident as reference PointBatch chunks (widened once)."""

    def __init__(self, vx, vy, xs32, ys32, threads: int | None = None):
        import oracle
        self.ref = oracle.Reference()
        self.kind = "reference"
        self.threads = threads or cores()
        self.vx, self.vy = np.asarray(vx, np.float64), np.asarray(vy, np.float64)
        self.m = int(xs32.size)
        self.chunks = self.ref.make_chunks(xs32, ys32, self.threads, CHUNK)

    def close(self):
        if self.chunks:
            self.ref.free_chunks(self.chunks)
            self.chunks = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def run(self, packed: bool = False):
        """Every point through the three reference engines: per engine
        {ns, count_ns, inside, words}; `ns` sums the batch calls only."""
        return self.ref.full_pass(self.vx, self.vy, None, None, self.threads, CHUNK,
                                  packed=packed, chunks=self.chunks, m=self.m)

    def describe(self) -> str:
        return (f"the unmodified reference library ({self.ref.build}), all {self.m} points of "
                f"the workload stream (f32 rounded, widened to f64) in PointBatch chunks of "
                f"{CHUNK} points, 3 engines *_contains_batch(threads={self.threads}) timed like "
                f"bench.cpp:196-199 and summed over the chunks; count_inside timed as its own step")


def band_outside(vx, vy, xs, ys, eps: float) -> np.ndarray:
    """True where a point lies farther than eps * max(1, |x|, |y|, polygon
    extent) from every edge's supporting line (edge_line_distance,
    voronoi.cpp:73-82): a disagreement there breaks parity."""
    import oracle
    orc = oracle.Oracle()
    xs = np.asarray(xs, np.float64)
    ys = np.asarray(ys, np.float64)
    if xs.size == 0:
        return np.zeros(0, bool)
    ext = max(np.ptp(vx), np.ptp(vy))
    s = np.maximum(np.maximum(1.0, np.abs(xs)), np.maximum(np.abs(ys), ext))
    with np.errstate(invalid="ignore"):
        return ~(orc.edge_line_distances(np.asarray(vx, float), np.asarray(vy, float), xs, ys)
                 <= eps * s)


def join_band_outside(off, vx, vy, xs, ys, ids, eps: float) -> np.ndarray:
    """band_outside for database pairs, each against its own polygon."""
    xs = np.asarray(xs, np.float64)
    ys = np.asarray(ys, np.float64)
    ids = np.asarray(ids, np.int64)
    out = np.zeros(xs.size, bool)
    for k in range(xs.size):
        i = ids[k]
        if i < 0 or i >= off.size - 1:
            continue
        a, b = int(off[i]), int(off[i + 1])
        out[k] = band_outside(vx[a:b], vy[a:b], xs[k:k + 1], ys[k:k + 1], eps)[0]
    return out


def diff_indices(words_a, words_b, m: int, limit: int = 1 << 20) -> np.ndarray:
    """Point indices where two LSB-first mask word arrays differ (torch CUDA
    tensors or numpy arrays; XORed where they live, only the differing words
    are brought back)."""
    try:
        import torch
        is_t = isinstance(words_a, torch.Tensor) or isinstance(words_b, torch.Tensor)
    except ImportError:
        is_t = False
    if is_t:
        dev = words_a.device if isinstance(words_a, torch.Tensor) else words_b.device
        ta = words_a if isinstance(words_a, torch.Tensor) else torch.as_tensor(
            np.asarray(words_a).view(np.int32), device=dev)
        tb = words_b if isinstance(words_b, torch.Tensor) else torch.as_tensor(
            np.asarray(words_b).view(np.int32), device=dev)
        x = torch.bitwise_xor(ta.view(torch.int32), tb.view(torch.int32))
        nz = torch.nonzero(x).flatten()[:limit]
        wi = nz.cpu().numpy().astype(np.int64)
        wv = x[nz].cpu().numpy().view(np.uint32)
    else:
        x = np.bitwise_xor(np.asarray(words_a).view(np.uint32), np.asarray(words_b).view(np.uint32))
        wi = np.flatnonzero(x)[:limit]
        wv = x[wi]
    bits = np.unpackbits(wv.view(np.uint8).reshape(-1, 4), axis=1, bitorder="little")
    idx = (wi[:, None] * 32 + np.arange(32)[None, :])[bits.astype(bool)]
    return idx[idx < m]


def parity_entry(words_gpu, words_ref, xs, ys, vx, vy, m: int, eps: float, join=None) -> dict:
    """{disagree, outside_band} of one engine's two masks over one batch."""
    idx = diff_indices(words_gpu, words_ref, m)
    px = np.asarray(xs[idx], np.float64) if idx.size else np.zeros(0)
    py = np.asarray(ys[idx], np.float64) if idx.size else np.zeros(0)
    if join is not None:
        off, ids = join
        out = join_band_outside(off, vx, vy, px, py, np.asarray(ids)[idx], eps)
    else:
        out = band_outside(vx, vy, px, py, eps)
    return {"disagree": int(idx.size), "outside_band": int(out.sum())}
