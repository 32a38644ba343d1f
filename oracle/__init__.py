"""CPU oracle for the B200 point-inclusion engine -- TEST INFRASTRUCTURE ONLY.

Two checkers, both loaded with ctypes:
  * `Oracle`    -- liboracle.so, the plain-C restatement of the reference path
                   (oracle/vpip_oracle.c, every function cites its reference
                   file:line), compiled with -ffp-contract=off;
  * `Reference` -- oracle/_ref/libvpip_ref.so, the UNMODIFIED reference sources
                   (/root/reference/proj/src) compiled by oracle/Makefile.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package, and only as the checker or the
CPU baseline -- never as the thing measured on the GPU path.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libvpip_ref.so"             # -march=x86-64-v3
REF_NATIVE_SO = HERE / "_ref" / "libvpip_ref_native.so"  # -march=<build host's native CPU>
REF_NATIVE_MARCH = HERE / "_ref" / "native_march.txt"
REF_ACCEPTANCE = HERE / "_ref" / "vpip_acceptance"
# the reference's acceptance suite linked against libvpipg (the drop-in check)
REF_ACCEPTANCE_B200 = HERE / "_ref" / "vpip_acceptance_b200"
# the reference's unit suites (on oracle/mini_doctest) against the reference / the drop-in
REF_UNIT = HERE / "_ref" / "vpip_unit_ref"
REF_UNIT_B200 = HERE / "_ref" / "vpip_unit_b200"
# the reference CLI (on oracle/mini_cli11) against the reference / the drop-in
REF_CLI = HERE / "_ref" / "vpip_cli_ref"
REF_CLI_B200 = HERE / "_ref" / "vpip_cli_b200"
REFERENCE_SRC = Path("/root/reference/proj")

_D = C.POINTER(C.c_double)
_U8 = C.POINTER(C.c_uint8)


def _d(a):
    return a.ctypes.data_as(_D)


def build(ref: bool | None = None) -> None:
    """Compile liboracle.so, and oracle/_ref when the reference tree is present."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if ref is None:
        ref = REFERENCE_SRC.exists()
    if ref:
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


class Oracle:
    """numpy-facing wrapper of the C restatement."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        sz = C.c_size_t
        L.vo_mix_seed.restype = C.c_uint64
        L.vo_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.vo_sample_points.argtypes = [sz, C.c_double, C.c_double, C.c_double, C.c_double,
                                       C.c_uint64, _D, _D]
        L.vo_regular_polygon.argtypes = [sz, C.c_double, C.c_double, C.c_double, _D, _D]
        L.vo_random_convex_polygon.argtypes = [sz, C.c_uint64, C.c_double, C.c_double,
                                               C.c_double, _D, _D]
        L.vo_validate_polygon.argtypes = [_D, _D, sz, C.c_double, C.POINTER(C.c_int)]
        L.vo_centroid.argtypes = [_D, _D, sz, _D, _D]
        L.vo_signed_area.restype = C.c_double
        L.vo_signed_area.argtypes = [_D, _D, sz]
        L.vo_edge_coefficients.argtypes = [C.c_double] * 4 + [_D]
        L.vo_reflect_generator.argtypes = [C.c_double, C.c_double, _D, _D, _D]
        L.vo_foot_of_perpendicular.argtypes = [C.c_double, C.c_double, _D, _D, _D]
        L.vo_to_voronoi.argtypes = [_D, _D, sz, _D, _D]
        L.vo_edge_line_distance.restype = C.c_double
        L.vo_edge_line_distance.argtypes = [_D, _D, sz, C.c_double, C.c_double]
        for f in ("vo_voronoi_batch",):
            getattr(L, f).argtypes = [_D, _D, sz, _D, _D, sz, _U8]
        for f in ("vo_offset_batch", "vo_ray_batch"):
            getattr(L, f).argtypes = [_D, _D, sz, _D, _D, sz, _U8]
        L.vo_voronoi_contains.argtypes = [_D, _D, sz, C.c_double, C.c_double]
        for f in ("vo_offset_contains", "vo_ray_contains", "vo_ray_count"):
            getattr(L, f).argtypes = [_D, _D, sz, C.c_double, C.c_double]
        L.vo_count_inside.restype = C.c_uint64
        L.vo_count_inside.argtypes = [_U8, sz]
        L.vo_pack_mask_lsb.argtypes = [_U8, sz, _U8]
        L.vo_counter_points_f32.argtypes = [C.c_uint64, C.c_uint64, sz, C.c_double, C.c_double,
                                            C.c_double, C.c_double, C.POINTER(C.c_float),
                                            C.POINTER(C.c_float)]
        u32p = C.POINTER(C.c_uint32)
        L.vo_join_pairs_f32.argtypes = [C.c_uint64, C.c_uint64, sz, C.c_uint32, _D, _D, _D,
                                        C.POINTER(C.c_float), C.POINTER(C.c_float), u32p]
        L.vo_csr_status.argtypes = [u32p, _D, _D, C.c_uint32, C.POINTER(C.c_int32)]
        L.vo_join_masks.argtypes = [u32p, _D, _D, C.c_uint32, C.c_int, _D, _D, u32p, sz, _U8]
        self.L = L

    # polygon-database join (config 4)
    def join_pairs_f32(self, seed, first, m, cx, cy, r):
        xs, ys = np.zeros(m, np.float32), np.zeros(m, np.float32)
        ids = np.zeros(m, np.uint32)
        fp, up = C.POINTER(C.c_float), C.POINTER(C.c_uint32)
        self.L.vo_join_pairs_f32(seed, first, m, len(cx), _d(np.ascontiguousarray(cx, np.float64)),
                                 _d(np.ascontiguousarray(cy, np.float64)),
                                 _d(np.ascontiguousarray(r, np.float64)),
                                 xs.ctypes.data_as(fp), ys.ctypes.data_as(fp), ids.ctypes.data_as(up))
        return xs, ys, ids

    def csr_status(self, offsets, vx, vy):
        offsets = np.ascontiguousarray(offsets, np.uint32)
        st = np.zeros(offsets.size - 1, np.int32)
        self.L.vo_csr_status(offsets.ctypes.data_as(C.POINTER(C.c_uint32)),
                             _d(np.ascontiguousarray(vx, np.float64)),
                             _d(np.ascontiguousarray(vy, np.float64)), offsets.size - 1,
                             st.ctypes.data_as(C.POINTER(C.c_int32)))
        return st

    def join_masks(self, offsets, vx, vy, engine, xs, ys, ids):
        offsets = np.ascontiguousarray(offsets, np.uint32)
        xs = np.ascontiguousarray(xs, np.float64)
        ys = np.ascontiguousarray(ys, np.float64)
        ids = np.ascontiguousarray(ids, np.uint32)
        out = np.zeros(xs.size, np.uint8)
        up = C.POINTER(C.c_uint32)
        self.L.vo_join_masks(offsets.ctypes.data_as(up), _d(np.ascontiguousarray(vx, np.float64)),
                             _d(np.ascontiguousarray(vy, np.float64)), offsets.size - 1, engine,
                             _d(xs), _d(ys), ids.ctypes.data_as(up), xs.size,
                             out.ctypes.data_as(_U8))
        return out

    # sampling
    def mix_seed(self, seed, salt):
        return self.L.vo_mix_seed(seed, salt)

    def sample_points(self, count, box, seed):
        xs, ys = np.zeros(count), np.zeros(count)
        rc = self.L.vo_sample_points(count, *map(float, box), seed, _d(xs), _d(ys))
        if rc:
            raise ValueError(rc)
        return xs, ys

    def regular_polygon(self, n, r=1.0, center=(0.0, 0.0)):
        vx, vy = np.zeros(n), np.zeros(n)
        rc = self.L.vo_regular_polygon(n, r, center[0], center[1], _d(vx), _d(vy))
        if rc:
            raise ValueError(rc)
        return vx, vy

    def random_convex_polygon(self, n, seed, r=1.0, center=(0.0, 0.0)):
        vx, vy = np.zeros(n), np.zeros(n)
        rc = self.L.vo_random_convex_polygon(n, seed, r, center[0], center[1], _d(vx), _d(vy))
        if rc:
            raise ValueError(rc)
        return vx, vy

    def counter_points_f32(self, seed, first, count, box):
        xs, ys = np.zeros(count, np.float32), np.zeros(count, np.float32)
        fp = C.POINTER(C.c_float)
        self.L.vo_counter_points_f32(seed, first, count, *map(float, box),
                                     xs.ctypes.data_as(fp), ys.ctypes.data_as(fp))
        return xs, ys

    # geometry / conversion
    def validate(self, vx, vy, eps=1e-12):
        vx, vy = np.array(vx, dtype=np.float64), np.array(vy, dtype=np.float64)
        rev = C.c_int()
        rc = self.L.vo_validate_polygon(_d(vx), _d(vy), vx.size, eps, C.byref(rev))
        return rc, vx, vy, bool(rev.value)

    def centroid(self, vx, vy):
        cx, cy = C.c_double(), C.c_double()
        self.L.vo_centroid(_d(vx), _d(vy), vx.size, C.byref(cx), C.byref(cy))
        return cx.value, cy.value

    def edge_coefficients(self, qi, qj):
        abc = np.zeros(3)
        rc = self.L.vo_edge_coefficients(qi[0], qi[1], qj[0], qj[1], _d(abc))
        return rc, abc

    def reflect(self, p, abc):
        rx, ry = C.c_double(), C.c_double()
        abc = np.asarray(abc, dtype=np.float64)
        rc = self.L.vo_reflect_generator(p[0], p[1], _d(abc), C.byref(rx), C.byref(ry))
        return rc, (rx.value, ry.value)

    def foot(self, p, abc):
        fx, fy = C.c_double(), C.c_double()
        abc = np.asarray(abc, dtype=np.float64)
        self.L.vo_foot_of_perpendicular(p[0], p[1], _d(abc), C.byref(fx), C.byref(fy))
        return fx.value, fy.value

    def to_voronoi(self, vx, vy):
        inner, outer = np.zeros(2), np.zeros((vx.size, 2))
        rc = self.L.vo_to_voronoi(_d(vx), _d(vy), vx.size, _d(inner), _d(outer))
        return rc, inner, outer

    def edge_line_distance(self, vx, vy, px, py):
        return self.L.vo_edge_line_distance(_d(vx), _d(vy), vx.size, px, py)

    def edge_line_distances(self, vx, vy, xs, ys):
        """Vectorised min over edges of |a x + b y + c| / hypot(a, b) (voronoi.cpp:73-82)."""
        xs = np.asarray(xs, dtype=np.float64)
        ys = np.asarray(ys, dtype=np.float64)
        d = np.full(xs.shape, np.inf)
        n = vx.size
        for k in range(n):
            k1 = (k + 1) % n
            a = vy[k] - vy[k1]
            b = vx[k1] - vx[k]
            c = -(a * vx[k] + b * vy[k])
            d = np.minimum(d, np.abs(a * xs + b * ys + c) / np.hypot(a, b))
        return d

    # engines
    def voronoi_batch(self, inner, outer, xs, ys):
        xs, ys = np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64)
        out = np.zeros(xs.size, np.uint8)
        inner = np.ascontiguousarray(inner, np.float64)
        outer = np.ascontiguousarray(outer, np.float64)
        self.L.vo_voronoi_batch(_d(inner), _d(outer), outer.shape[0], _d(xs), _d(ys), xs.size,
                                out.ctypes.data_as(_U8))
        return out

    def offset_batch(self, vx, vy, xs, ys):
        xs, ys = np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64)
        out = np.zeros(xs.size, np.uint8)
        self.L.vo_offset_batch(_d(vx), _d(vy), vx.size, _d(xs), _d(ys), xs.size,
                               out.ctypes.data_as(_U8))
        return out

    def ray_batch(self, vx, vy, xs, ys):
        xs, ys = np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64)
        vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
        out = np.zeros(xs.size, np.uint8)
        self.L.vo_ray_batch(_d(vx), _d(vy), vx.size, _d(xs), _d(ys), xs.size,
                            out.ctypes.data_as(_U8))
        return out

    def masks(self, vx_raw, vy_raw, xs, ys):
        """All three engines the way the reference CLI builds them (vpip.cpp:120-133)."""
        rc, vx, vy, _ = self.validate(vx_raw, vy_raw)
        if rc:
            raise ValueError(rc)
        rc, inner, outer = self.to_voronoi(vx, vy)
        if rc:
            raise ValueError(rc)
        return (self.voronoi_batch(inner, outer, xs, ys), self.offset_batch(vx, vy, xs, ys),
                self.ray_batch(np.asarray(vx_raw, np.float64), np.asarray(vy_raw, np.float64),
                               xs, ys))

    def pack(self, mask):
        mask = np.ascontiguousarray(mask, np.uint8)
        out = np.zeros((mask.size + 7) // 8, np.uint8)
        self.L.vo_pack_mask_lsb(mask.ctypes.data_as(_U8), mask.size, out.ctypes.data_as(_U8))
        return out


def native_march() -> str | None:
    """What `-march=native` resolves to on this host (gcc), e.g. 'sapphirerapids'."""
    try:
        out = subprocess.run(["gcc", "-march=native", "-Q", "--help=target"], capture_output=True,
                             text=True, timeout=30).stdout
    except Exception:
        return None
    for line in out.splitlines():
        parts = line.split()
        if parts and parts[0] == "-march=" and len(parts) > 1:
            return parts[1]
    return None


class Reference:
    """The unmodified reference library (oracle/_ref/libvpip_ref*.so).

    Loads the -march=native build when this host's native CPU is the one it
    was built for (the reference's Release flags, CMakeLists.txt:13-17),
    else the portable x86-64-v3 build; `self.build` says which."""

    def __init__(self, native: bool = True):
        so, self.build = REF_SO, "-O3 -DNDEBUG -march=x86-64-v3 -ffp-contract=off"
        if native and REF_NATIVE_SO.exists() and REF_NATIVE_MARCH.exists():
            built = REF_NATIVE_MARCH.read_text().strip()
            here = native_march()
            if built and built == here:
                so = REF_NATIVE_SO
                self.build = (f"-O3 -DNDEBUG -march={built} -ffp-contract=off "
                              f"(= -march=native on this host)")
        if not so.exists():
            raise FileNotFoundError(f"{so} not built (needs /root/reference; run oracle.build())")
        L = C.CDLL(str(so))
        sz = C.c_size_t
        L.vr_validate.argtypes = [_D, _D, sz, _D, _D, C.POINTER(C.c_int)]
        L.vr_to_voronoi.argtypes = [_D, _D, sz, _D, _D]
        L.vr_edge_coefficients.argtypes = [C.c_double] * 4 + [_D]
        L.vr_reflect_generator.argtypes = [C.c_double, C.c_double, _D, _D]
        L.vr_edge_line_distance.restype = C.c_double
        L.vr_edge_line_distance.argtypes = [_D, _D, sz, C.c_double, C.c_double]
        L.vr_mix_seed.restype = C.c_uint64
        L.vr_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.vr_sample_points.argtypes = [sz, C.c_double, C.c_double, C.c_double, C.c_double,
                                       C.c_uint64, _D, _D]
        L.vr_regular_polygon.argtypes = [sz, C.c_double, C.c_double, C.c_double, _D, _D]
        L.vr_random_convex_polygon.argtypes = [sz, C.c_uint64, C.c_double, C.c_double,
                                               C.c_double, _D, _D]
        L.vr_batch_new.restype = C.c_void_p
        L.vr_batch_new.argtypes = [_D, _D, sz]
        L.vr_batch_free.argtypes = [C.c_void_p]
        L.vr_poly_new.restype = C.c_void_p
        L.vr_poly_new.argtypes = [_D, _D, sz, C.c_int, C.POINTER(C.c_int)]
        L.vr_poly_free.argtypes = [C.c_void_p]
        L.vr_run_engine.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, _U8,
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.vr_voronoi_batch_gens.argtypes = [_D, _D, sz, C.c_void_p, C.c_int, _U8,
                                            C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.vr_scalar.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double]
        L.vr_run_validation.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                        C.POINTER(C.c_uint64)]
        L.vr_read_bench_csv.restype = C.c_long
        L.vr_read_bench_csv.argtypes = [C.c_char_p, _D]
        u32p = C.POINTER(C.c_uint32)
        L.vr_join_new.restype = C.c_void_p
        L.vr_join_new.argtypes = [u32p, _D, _D, C.c_uint32, _D, _D, u32p, sz]
        L.vr_join_free.argtypes = [C.c_void_p]
        L.vr_join_run.restype = C.c_uint64
        L.vr_join_run.argtypes = [C.c_void_p, C.c_int, C.c_int, _U8]
        L.vr_join_scalar.restype = C.c_uint64
        L.vr_join_scalar.argtypes = [C.c_void_p, _D, _D, u32p, sz, C.c_int, C.c_int, _U8]
        fp = C.POINTER(C.c_float)
        L.vr_time_convert.argtypes = [_D, _D, sz, C.c_int, C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64)]
        L.vr_time_convert_csr.argtypes = [C.POINTER(C.c_uint32), _D, _D, C.c_uint32,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.vr_chunks_new.restype = C.c_void_p
        L.vr_chunks_new.argtypes = [fp, fp, sz, sz, C.c_int]
        L.vr_chunks_free.argtypes = [C.c_void_p]
        u64p = C.POINTER(C.c_uint64)
        L.vr_chunked_run.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, _U8, u64p, u64p, u64p]
        self.L = L

    def read_bench_csv(self, text: str):
        """The reference's read_bench_csv + median: (#records, medians[3][13] for n=3..15)."""
        med = np.zeros(39)
        n = self.L.vr_read_bench_csv(text.encode(), _d(med))
        return n, med.reshape(3, 13)

    def run_validation(self, vx, vy, xs, ys, band=1e-9, threads=1):
        """The reference's run_validation: ({pair counts}, disagreeing, pass)."""
        vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
        xs, ys = np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64)
        code = C.c_int()
        p = self.L.vr_poly_new(_d(vx), _d(vy), vx.size, 1, C.byref(code))
        if not p:
            raise ValueError(code.value)
        b = self.L.vr_batch_new(_d(xs), _d(ys), xs.size)
        out = (C.c_uint64 * 5)()
        try:
            self.L.vr_run_validation(p, b, threads, band, out)
        finally:
            self.L.vr_batch_free(b)
            self.L.vr_poly_free(p)
        return list(out[:3]), out[3], bool(out[4])

    def join(self, offsets, vx, vy, xs, ys, ids, threads=1, engines=(0, 1, 2)):
        """Per-polygon batch calls over id-grouped pairs (grouping untimed).
        Returns (masks, ns per engine)."""
        offsets = np.ascontiguousarray(offsets, np.uint32)
        xs, ys = np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64)
        ids = np.ascontiguousarray(ids, np.uint32)
        up = C.POINTER(C.c_uint32)
        h = self.L.vr_join_new(offsets.ctypes.data_as(up), _d(np.ascontiguousarray(vx, np.float64)),
                               _d(np.ascontiguousarray(vy, np.float64)), offsets.size - 1,
                               _d(xs), _d(ys), ids.ctypes.data_as(up), xs.size)
        out, times = [], []
        try:
            for e in engines:
                m = np.zeros(xs.size, np.uint8)
                times.append(self.L.vr_join_run(h, e, threads, m.ctypes.data_as(_U8)))
                out.append(m)
        finally:
            self.L.vr_join_free(h)
        return out, times

    def join_scalar(self, offsets, vx, vy, xs, ys, ids, engine, threads=1):
        """The per-pair scalar join loop (pairs in stream order). Returns (mask, ns)."""
        offsets = np.ascontiguousarray(offsets, np.uint32)
        xs, ys = np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64)
        ids = np.ascontiguousarray(ids, np.uint32)
        up = C.POINTER(C.c_uint32)
        h = self.L.vr_join_new(offsets.ctypes.data_as(up), _d(np.ascontiguousarray(vx, np.float64)),
                               _d(np.ascontiguousarray(vy, np.float64)), offsets.size - 1,
                               _d(xs[:0]), _d(ys[:0]), ids.ctypes.data_as(up), 0)
        m = np.zeros(xs.size, np.uint8)
        try:
            ns = self.L.vr_join_scalar(h, _d(xs), _d(ys), ids.ctypes.data_as(up), xs.size, engine,
                                       threads, m.ctypes.data_as(_U8))
        finally:
            self.L.vr_join_free(h)
        return m, ns

    def full_pass(self, vx, vy, xs32, ys32, threads, chunk=1 << 26, engines=(0, 1, 2),
                  packed=True, chunks=None, m=None):
        """Every point of an f32 workload through the reference in <= `chunk`-point
        PointBatches (widened once, untimed). Returns per engine
        {ns, count_ns, inside, words (LSB-first u32 mask words or None)}.
        `chunks` reuses a handle from `make_chunks` (the caller frees it)."""
        vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
        code = C.c_int()
        p = self.L.vr_poly_new(_d(vx), _d(vy), vx.size, 1 if any(e != 2 for e in engines) else 0,
                               C.byref(code))
        if not p:
            raise ValueError(code.value)
        own = chunks is None
        if own:
            chunks = self.make_chunks(xs32, ys32, threads, chunk)
        m = int(np.asarray(xs32).size) if m is None else m
        res = []
        try:
            for e in engines:
                words = np.zeros((m + 31) // 32, np.uint32) if packed else None
                ns, cns, ins = C.c_uint64(), C.c_uint64(), C.c_uint64()
                rc = self.L.vr_chunked_run(p, chunks, e, threads,
                                           words.view(np.uint8).ctypes.data_as(_U8) if packed else None,
                                           C.byref(ns), C.byref(cns), C.byref(ins))
                if rc:
                    raise ValueError(rc)
                res.append({"ns": ns.value, "count_ns": cns.value, "inside": ins.value,
                            "words": words})
        finally:
            self.L.vr_poly_free(p)
            if own:
                self.free_chunks(chunks)
        return res

    def time_convert(self, vx, vy, reps=101):
        """Medians (ns) of validate_polygon and of to_voronoi (bench.cpp:165-170)."""
        vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
        tv, tc = C.c_uint64(), C.c_uint64()
        rc = self.L.vr_time_convert(_d(vx), _d(vy), vx.size, reps, C.byref(tv), C.byref(tc))
        if rc:
            raise ValueError(rc)
        return tv.value, tc.value

    def time_convert_csr(self, offsets, vx, vy):
        """Total ns of validate_polygon and to_voronoi over a CSR database (1 thread)."""
        offsets = np.ascontiguousarray(offsets, np.uint32)
        tv, tc = C.c_uint64(), C.c_uint64()
        self.L.vr_time_convert_csr(offsets.ctypes.data_as(C.POINTER(C.c_uint32)),
                                   _d(np.ascontiguousarray(vx, np.float64)),
                                   _d(np.ascontiguousarray(vy, np.float64)), offsets.size - 1,
                                   C.byref(tv), C.byref(tc))
        return tv.value, tc.value

    def make_chunks(self, xs32, ys32, threads, chunk=1 << 26):
        xs32 = np.ascontiguousarray(xs32, np.float32)
        ys32 = np.ascontiguousarray(ys32, np.float32)
        fp = C.POINTER(C.c_float)
        return self.L.vr_chunks_new(xs32.ctypes.data_as(fp), ys32.ctypes.data_as(fp), xs32.size,
                                    chunk, threads)

    def free_chunks(self, h):
        self.L.vr_chunks_free(h)

    def validate(self, vx, vy):
        vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
        ox, oy = np.zeros(vx.size), np.zeros(vx.size)
        rev = C.c_int()
        rc = self.L.vr_validate(_d(vx), _d(vy), vx.size, _d(ox), _d(oy), C.byref(rev))
        return rc, ox, oy, bool(rev.value)

    def to_voronoi(self, vx, vy):
        vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
        inner, outer = np.zeros(2), np.zeros((vx.size, 2))
        rc = self.L.vr_to_voronoi(_d(vx), _d(vy), vx.size, _d(inner), _d(outer))
        return rc, inner, outer

    def sample_points(self, count, box, seed):
        xs, ys = np.zeros(count), np.zeros(count)
        rc = self.L.vr_sample_points(count, *map(float, box), seed, _d(xs), _d(ys))
        if rc:
            raise ValueError(rc)
        return xs, ys

    def regular_polygon(self, n, r=1.0, center=(0.0, 0.0)):
        vx, vy = np.zeros(n), np.zeros(n)
        rc = self.L.vr_regular_polygon(n, r, center[0], center[1], _d(vx), _d(vy))
        if rc:
            raise ValueError(rc)
        return vx, vy

    def random_convex_polygon(self, n, seed, r=1.0, center=(0.0, 0.0)):
        vx, vy = np.zeros(n), np.zeros(n)
        rc = self.L.vr_random_convex_polygon(n, seed, r, center[0], center[1], _d(vx), _d(vy))
        if rc:
            raise ValueError(rc)
        return vx, vy

    def masks(self, vx, vy, xs, ys, threads=1, engines=(0, 1, 2)):
        """Masks of the requested engines (0 voronoi, 1 offset, 2 crossing) + timings (ns)."""
        vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
        xs, ys = np.ascontiguousarray(xs, np.float64), np.ascontiguousarray(ys, np.float64)
        code = C.c_int()
        p = self.L.vr_poly_new(_d(vx), _d(vy), vx.size, 1 if any(e != 2 for e in engines) else 0,
                               C.byref(code))
        if not p:
            raise ValueError(code.value)
        b = self.L.vr_batch_new(_d(xs), _d(ys), xs.size)
        out, times = [], []
        try:
            for e in engines:
                m = np.zeros(xs.size, np.uint8)
                ns = C.c_uint64()
                self.L.vr_run_engine(p, e, b, threads, m.ctypes.data_as(_U8), C.byref(ns), None)
                out.append(m)
                times.append(ns.value)
        finally:
            self.L.vr_batch_free(b)
            self.L.vr_poly_free(p)
        return out, times
