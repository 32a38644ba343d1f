"""Python host mirror of the vpip engine interface over the C-ABI.

`PreparedPolygon` is the handle of include/vpipg.h (vpipg_prepare /
vpipg_prepare_generators); `test()` is the fused batch test + count
(vpipg_test) on device tensors, `test_host()` the host-buffer drop-in
(vpipg_test_host). Names and argument meaning follow the reference API
(proj/include/vpip/engines.hpp, voronoi.hpp); errors raise VpipError with the
reference's ErrorCode. torch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (ENGINES, F32, F64, KIND_ALL, KIND_CROSSING, KIND_OFFSET, KIND_VORONOI,
                   VpipError, check, load)

__all__ = ["PreparedPolygon", "PolygonDB", "fill_join_pairs", "VpipError", "fill_uniform_points", "mix_seed",
           "regular_polygon", "random_convex_polygon", "sample_points", "KIND_ALL",
           "KIND_VORONOI", "KIND_OFFSET", "KIND_CROSSING", "F32", "F64"]


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _stream_ptr(stream) -> C.c_void_p:
    if stream is None:
        return C.c_void_p(None)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)  # torch.cuda.Stream


def _out_specs(m, words=None, bytes_=None, count=None):
    """(tensor, minimum numel, kind) for the output checks of _check_device_batch."""
    return [(words, (m + 31) // 32, "words"), (bytes_, m, "bytes"), (count, 1, "count")]


def _check_device_batch(xs, ys, dtypes, outs=(), ids=None, device=None) -> None:
    """The C-ABI takes raw pointers; the Python mirror checks what it can see
    (vpip::Error InvalidParameter, code 6, on a mismatch): inputs 1-D,
    contiguous, same length and dtype; every tensor on the handle's GPU; mask
    words 4-byte elements, byte masks 1-byte elements, counters 64-bit integers
    (the kernels atomically add a u64), each large enough."""
    import torch
    m = xs.numel()
    ok = (xs.is_cuda and ys.is_cuda and xs.dtype in dtypes and ys.dtype == xs.dtype
          and ys.numel() == m and xs.is_contiguous() and ys.is_contiguous())
    tensors = [xs, ys]
    if ids is not None:
        ok = ok and ids.is_cuda and ids.numel() == m and ids.is_contiguous() and \
            ids.element_size() == 4
        tensors.append(ids)
    for t, need, kind in outs:
        if t is None:
            continue
        tensors.append(t)
        ok = ok and t.is_cuda and t.is_contiguous() and t.numel() >= need
        if kind == "words":
            ok = ok and t.element_size() == 4 and not t.is_floating_point()
        elif kind == "bytes":
            ok = ok and t.element_size() == 1 and not t.is_floating_point()
        else:
            ok = ok and t.dtype in (torch.int64, getattr(torch, "uint64", torch.int64))
    if ok and device is not None:
        ok = all(t.device.index == device for t in tensors)
    if not ok:
        raise VpipError(6, "device batch: 1-D contiguous CUDA tensors of matching length "
                           "and dtype on the handle's device, int32 mask words, uint8 byte "
                           "masks and int64 counters of sufficient size are required")


def _host_view(a):
    """(dtype name, numel, 1-D contiguous host buffer, element size) of a numpy
    array or a CPU torch tensor; None for anything else."""
    if isinstance(a, np.ndarray):
        return a.dtype.name, a.size, a.ndim == 1 and a.flags.c_contiguous, a.itemsize
    if hasattr(a, "is_cuda") and hasattr(a, "element_size"):
        return (str(a.dtype).rsplit(".", 1)[-1], a.numel(),
                a.dim() == 1 and a.is_contiguous() and not a.is_cuda, a.element_size())
    return None


def _check_host_batch(xs, ys, dtypes, ids=None, words=None) -> None:
    """The host-buffer calls read m elements of xs / ys (/ ids) and write
    ceil(m/32) words per engine through raw pointers, so the mirror checks what
    the C-ABI cannot see (InvalidParameter, code 6): 1-D contiguous host
    buffers of one floating dtype and one length, 4-byte integer ids, and
    caller-provided word buffers of 4-byte elements large enough for the batch."""
    vx, vy = _host_view(xs), _host_view(ys)
    ok = (vx is not None and vy is not None and vx[2] and vy[2] and vx[0] in dtypes
          and vy[0] == vx[0] and vy[1] == vx[1])
    m = vx[1] if ok else 0
    if ok and ids is not None:
        vi = _host_view(ids)
        ok = vi is not None and vi[2] and vi[1] == m and vi[0] in ("int32", "uint32")
    for w in (words or ()):
        if w is None or not ok:
            continue
        vw = _host_view(w)
        ok = (vw is not None and vw[2] and vw[3] == 4 and vw[0] in ("int32", "uint32")
              and vw[1] >= (m + 31) // 32)
    if not ok:
        raise VpipError(6, "host batch: 1-D contiguous host buffers (numpy or CPU tensors) of "
                           f"matching length and dtype ({', '.join(dtypes)}), 32-bit ids and "
                           "32-bit mask-word buffers of ceil(m/32) elements are required")


def _engine_id(engine) -> int:
    return ENGINES[engine] if isinstance(engine, str) else int(engine)


class PreparedPolygon:
    """A polygon converted on the device (validate_polygon + to_voronoi + edge tables)."""

    def __init__(self, handle: C.c_void_p, n: int, device: int = 0):
        self._h = handle
        self.n = n
        self.device = device

    @classmethod
    def prepare(cls, vx, vy, kinds: int = KIND_ALL, device: int = 0, stream=None):
        vx = np.ascontiguousarray(vx, dtype=np.float64)
        vy = np.ascontiguousarray(vy, dtype=np.float64)
        if vx.shape != vy.shape or vx.ndim != 1:
            raise VpipError(6, "prepare")
        h = C.c_void_p()
        check(load().vpipg_prepare(_dptr(vx), _dptr(vy), vx.size, kinds, device,
                                   _stream_ptr(stream), C.byref(h)), "vpipg_prepare")
        return cls(h, vx.size, device)

    @classmethod
    def from_generators(cls, inner, outer, device: int = 0, stream=None):
        inner = np.ascontiguousarray(inner, dtype=np.float64).reshape(2)
        outer = np.ascontiguousarray(outer, dtype=np.float64).reshape(-1, 2)
        h = C.c_void_p()
        check(load().vpipg_prepare_generators(_dptr(inner), _dptr(outer), outer.shape[0], device,
                                              _stream_ptr(stream), C.byref(h)),
              "vpipg_prepare_generators")
        return cls(h, outer.shape[0], device)

    def close(self) -> None:
        if self._h:
            load().vpipg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def info(self):
        n, kinds, rev = C.c_uint32(), C.c_uint32(), C.c_int()
        check(load().vpipg_poly_info(self._h, C.byref(n), C.byref(kinds), C.byref(rev)))
        return n.value, kinds.value, bool(rev.value)

    def generators(self):
        """(inner[2], outer[n, 2]) as built on the device (GeneratorSet)."""
        inner = np.zeros(2)
        outer = np.zeros((self.n, 2))
        check(load().vpipg_poly_generators(self._h, _dptr(inner), _dptr(outer)), "generators")
        return inner, outer

    def vertices(self):
        vx, vy = np.zeros(self.n), np.zeros(self.n)
        check(load().vpipg_poly_vertices(self._h, _dptr(vx), _dptr(vy)))
        return vx, vy

    def test(self, engine, xs, ys, words=None, bytes_=None, count=None, stream=None) -> None:
        """Fused batch test on device tensors (vpipg_test). Asynchronous.

        xs, ys: 1-D CUDA tensors (float32 -> F32 kernels, float64 -> exact F64
        kernels). words: int32 tensor of ceil(m/32) (PIPM bit order); bytes_:
        uint8 tensor of m; count: int64 tensor of 1 (accumulated).
        """
        import torch
        m = xs.numel()
        _check_device_batch(xs, ys, (torch.float32, torch.float64),
                            _out_specs(m, words, bytes_, count), device=self.device)
        dtype = F32 if xs.dtype == torch.float32 else F64
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(None)
        check(load().vpipg_test(self._h, _engine_id(engine), dtype, ptr(xs), ptr(ys), m,
                                ptr(words), ptr(bytes_), ptr(count), _stream_ptr(stream)),
              "vpipg_test")

    def multi_fused(self, xs, ys, engines=(0, 1, 2)) -> bool:
        """Whether test_multi runs this batch as one fused kernel (vpipg_test_multi_fused)."""
        return self.multi_route(xs, ys, engines) != 0

    def multi_route(self, xs, ys, engines=(0, 1, 2)) -> int:
        """vpipg_test_multi_fused's answer: 0 one engine at a time, 1 a general
        fused kernel, 2 the small-polygon kernel (word outputs only)."""
        import torch
        mask = 0
        for e in engines:
            mask |= 1 << _engine_id(e)
        dtype = F32 if xs.dtype == torch.float32 else F64
        return int(load().vpipg_test_multi_fused(self._h, mask, dtype, C.c_void_p(xs.data_ptr()),
                                                 C.c_void_p(ys.data_ptr()), xs.numel()))

    def test_multi(self, xs, ys, engines=(0, 1, 2), words=None, bytes_=None, counts=None,
                   stream=None) -> None:
        """Several engines over one device batch (vpipg_test_multi): words /
        bytes_ / counts are lists of 3 (entries may be None; counts entries are
        int64 tensors of 1, accumulated). All three engines on float32 points
        run as one fused kernel. Asynchronous."""
        import torch
        m = xs.numel()
        outs = []
        for e in range(3):
            pick = lambda lst: lst[e] if lst is not None and e < len(lst) else None
            outs += _out_specs(m, pick(words), pick(bytes_), pick(counts))
        _check_device_batch(xs, ys, (torch.float32, torch.float64), outs, device=self.device)
        mask = 0
        for e in engines:
            mask |= 1 << _engine_id(e)
        arr = lambda lst: (C.c_void_p * 3)(*[C.c_void_p(t.data_ptr() if t is not None else None)
                                             for t in (lst or [None] * 3)])
        dtype = F32 if xs.dtype == torch.float32 else F64
        check(load().vpipg_test_multi(self._h, mask, dtype, C.c_void_p(xs.data_ptr()),
                                      C.c_void_p(ys.data_ptr()), m, arr(words), arr(bytes_),
                                      arr(counts), _stream_ptr(stream)), "vpipg_test_multi")

    def test_host(self, engine, xs: np.ndarray, ys: np.ndarray, words: bool = True,
                  bytes_: bool = False):
        """Host-buffer drop-in (vpipg_test_host): returns (words|None, bytes|None, count)."""
        _check_host_batch(xs, ys, ("float32", "float64"))
        dtype = F32 if xs.dtype == np.float32 else F64
        m = xs.size
        w = np.zeros((m + 31) // 32, dtype=np.uint32) if words else None
        b = np.zeros(m, dtype=np.uint8) if bytes_ else None
        cnt = C.c_uint64()
        vp = lambda a: C.c_void_p(a.ctypes.data) if a is not None else C.c_void_p(None)
        check(load().vpipg_test_host(self._h, _engine_id(engine), dtype, vp(xs), vp(ys), m,
                                     vp(w), vp(b), C.byref(cnt)), "vpipg_test_host")
        return w, b, cnt.value


    def validate(self, xs, ys, band: float = 1e-9, relative: bool = False, stream=None):
        """run_validation on the device (vpipg_validate): returns a dict report."""
        import torch
        _check_device_batch(xs, ys, (torch.float32, torch.float64), device=self.device)
        rep = _lib.Report()
        dtype = F32 if xs.dtype == torch.float32 else F64
        check(load().vpipg_validate(self._h, dtype, C.c_void_p(xs.data_ptr()),
                                    C.c_void_p(ys.data_ptr()), xs.numel(), band, int(relative),
                                    C.byref(rep), _stream_ptr(stream)), "vpipg_validate")
        return _report_dict(rep)

    def compare_masks(self, xs, ys, words_a, words_b, band: float, relative: bool = True,
                      stream=None):
        """Band classification of two masks of one batch (vpipg_compare_masks)."""
        import torch
        m = xs.numel()
        _check_device_batch(xs, ys, (torch.float32, torch.float64),
                            _out_specs(m, words_a) + _out_specs(m, words_b), device=self.device)
        rep = _lib.Report()
        dtype = F32 if xs.dtype == torch.float32 else F64
        check(load().vpipg_compare_masks(self._h, dtype, C.c_void_p(xs.data_ptr()),
                                         C.c_void_p(ys.data_ptr()), xs.numel(),
                                         C.c_void_p(words_a.data_ptr()),
                                         C.c_void_p(words_b.data_ptr()), band, int(relative),
                                         C.byref(rep), _stream_ptr(stream)), "vpipg_compare_masks")
        return _report_dict(rep)

    def test_host_multi(self, xs: np.ndarray, ys: np.ndarray, engines=(0, 1, 2),
                        words=None, counts_only: bool = False):
        """All requested engines over one host batch (vpipg_test_host_multi).

        `words`: optional list of 3 preallocated uint32 arrays (e.g. pinned
        buffers); returns (words list, counts list)."""
        _check_host_batch(xs, ys, ("float32", "float64"), words=words)
        is_np = isinstance(xs, np.ndarray)
        dtype = F32 if str(xs.dtype).endswith("float32") else F64
        m = xs.size if is_np else xs.numel()
        mask = 0
        for e in engines:
            mask |= 1 << _engine_id(e)
        if words is None and not counts_only:
            words = [np.zeros((m + 31) // 32, dtype=np.uint32) if (mask >> e) & 1 else None
                     for e in range(3)]
        wp = (C.c_void_p * 3)(*[C.c_void_p(w.ctypes.data if isinstance(w, np.ndarray) else
                                           (w.data_ptr() if w is not None else None))
                                for w in (words or [None] * 3)])
        cnt = (C.c_uint64 * 3)()
        check(load().vpipg_test_host_multi(self._h, mask, dtype, C.c_void_p(_host_ptr(xs)),
                                           C.c_void_p(_host_ptr(ys)), m, wp, None, cnt),
              "vpipg_test_host_multi")
        return words, [cnt[i] for i in range(3)]


class PolygonDB:
    """A CSR batch of polygons prepared on the device (vpipg_prepare_csr)."""

    def __init__(self, handle: C.c_void_p, npoly: int, status: np.ndarray, device: int = 0,
                 offsets: np.ndarray | None = None):
        self._h = handle
        self.offsets = offsets
        self.npoly = npoly
        self.status = status
        self.device = device

    @classmethod
    def prepare(cls, offsets, vx, vy, kinds: int = KIND_ALL, device: int = 0, stream=None):
        offsets = np.ascontiguousarray(offsets, dtype=np.uint32)
        vx = np.ascontiguousarray(vx, dtype=np.float64)
        vy = np.ascontiguousarray(vy, dtype=np.float64)
        npoly = offsets.size - 1
        # the C-ABI checks that offsets start at 0 and never decrease, but it
        # cannot see the vertex arrays' length: it reads offsets[-1] of each
        if (offsets.ndim != 1 or npoly < 0 or vx.ndim != 1 or vx.shape != vy.shape
                or int(offsets[-1]) > vx.size):
            raise VpipError(6, "prepare_csr: 1-D offsets of npoly + 1 entries whose last entry "
                               "does not exceed the length of vx == length of vy")
        status = np.zeros(max(npoly, 1), dtype=np.int32)
        h = C.c_void_p()
        check(load().vpipg_prepare_csr(C.c_void_p(offsets.ctypes.data), _dptr(vx), _dptr(vy),
                                       npoly, kinds, device, _stream_ptr(stream), C.byref(h),
                                       C.c_void_p(status.ctypes.data)), "vpipg_prepare_csr")
        return cls(h, npoly, status[:npoly], device, offsets.copy())

    def close(self) -> None:
        if self._h:
            load().vpipg_db_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def generators(self, poly: int, n: int | None = None):
        """(inner[2], outer[n, 2]) of polygon `poly`; n is its vertex count
        (taken from the offsets; a caller's n must agree with it)."""
        if not 0 <= poly < self.npoly or self.offsets is None:
            raise VpipError(6, "generators: polygon index out of range (or no offsets)")
        size = int(self.offsets[poly + 1]) - int(self.offsets[poly])
        if n is not None and n != size:
            raise VpipError(6, f"generators: polygon {poly} has {size} vertices, not {n}")
        inner, outer = np.zeros(2), np.zeros((size, 2))
        check(load().vpipg_db_generators(self._h, poly, _dptr(inner), _dptr(outer)), "generators")
        return inner, outer

    def test(self, engine, xs, ys, ids, words=None, bytes_=None, count=None, stream=None) -> None:
        """Gathered test on device tensors (vpipg_test_gather); float32 points, int32 ids."""
        import torch
        m = xs.numel()
        _check_device_batch(xs, ys, (torch.float32,), _out_specs(m, words, bytes_, count), ids=ids,
                            device=self.device)
        ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(None)
        check(load().vpipg_test_gather(self._h, _engine_id(engine), ptr(xs), ptr(ys), ptr(ids),
                                       xs.numel(), ptr(words), ptr(bytes_), ptr(count),
                                       _stream_ptr(stream)), "vpipg_test_gather")

    def test_multi(self, xs, ys, ids, engines=(0, 1, 2), words=None, bytes_=None, counts=None,
                   stream=None) -> None:
        """Several engines over one batch of device pairs (vpipg_test_gather_multi):
        words / bytes_ / counts are lists of 3 (entries may be None). All three
        engines run as one fused kernel. Asynchronous."""
        import torch
        m = xs.numel()
        outs = []
        for e in range(3):
            pick = lambda lst: lst[e] if lst is not None and e < len(lst) else None
            outs += _out_specs(m, pick(words), pick(bytes_), pick(counts))
        _check_device_batch(xs, ys, (torch.float32,), outs, ids=ids, device=self.device)
        mask = 0
        for e in engines:
            mask |= 1 << _engine_id(e)
        arr = lambda lst: (C.c_void_p * 3)(*[C.c_void_p(t.data_ptr() if t is not None else None)
                                             for t in (lst or [None] * 3)])
        check(load().vpipg_test_gather_multi(self._h, mask, C.c_void_p(xs.data_ptr()),
                                             C.c_void_p(ys.data_ptr()), C.c_void_p(ids.data_ptr()),
                                             m, arr(words), arr(bytes_), arr(counts),
                                             _stream_ptr(stream)), "vpipg_test_gather_multi")

    def test_host(self, xs, ys, ids, engines=(0, 1, 2), words=None, counts_only: bool = False):
        """The join over host buffers (vpipg_test_gather_host): float32 xs / ys and
        uint32 / int32 ids, numpy arrays or (pinned) CPU tensors. Returns
        (words list, counts list)."""
        _check_host_batch(xs, ys, ("float32",), ids=ids, words=words)
        m = xs.size if isinstance(xs, np.ndarray) else xs.numel()
        mask = 0
        for e in engines:
            mask |= 1 << _engine_id(e)
        if words is None and not counts_only:
            words = [np.zeros((m + 31) // 32, dtype=np.uint32) if (mask >> e) & 1 else None
                     for e in range(3)]
        wp = (C.c_void_p * 3)(*[C.c_void_p(_host_ptr(w) if w is not None else None)
                                for w in (words or [None] * 3)])
        cnt = (C.c_uint64 * 3)()
        check(load().vpipg_test_gather_host(self._h, mask, C.c_void_p(_host_ptr(xs)),
                                            C.c_void_p(_host_ptr(ys)), C.c_void_p(_host_ptr(ids)),
                                            m, wp, None, cnt), "vpipg_test_gather_host")
        return words, [cnt[i] for i in range(3)]


def fill_join_pairs(seed: int, first: int, xs, ys, ids, cx, cy, r, stream=None) -> None:
    """Join-pair generator on the device (vpipg_fill_join_pairs); cx, cy, r: CUDA f64."""
    ptr = lambda t: C.c_void_p(t.data_ptr())
    check(load().vpipg_fill_join_pairs(seed, first, xs.numel(), cx.numel(), ptr(cx), ptr(cy),
                                       ptr(r), ptr(xs), ptr(ys), ptr(ids), _stream_ptr(stream)),
          "fill_join_pairs")


def _report_dict(rep) -> dict:
    k = rep.n_samples
    return {"point_count": rep.point_count, "pair_disagreements": list(rep.pair_disagreements),
            "disagreeing_points": rep.disagreeing_points, "outside_band": rep.outside_band,
            "pass": bool(rep.pass_), "sample_index": list(rep.sample_index[:k]),
            "sample_dist": list(rep.sample_dist[:k]), "sample_engines": list(rep.sample_engines[:k])}


def _host_ptr(a) -> int:
    return a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()


def release_staging(device: int = 0) -> None:
    """Free the per-device staging the host-buffer calls keep (vpipg_release_staging)."""
    check(load().vpipg_release_staging(device), "vpipg_release_staging")


def zero_counts(counts, stream=None) -> None:
    """Zero a device int64 / uint64 counter tensor on `stream` with a memset
    (vpipg_zero_counts): no kernel launch, graph-capturable."""
    if not (counts.is_cuda and counts.is_contiguous() and counts.element_size() == 8):
        raise VpipError(6, "zero_counts: a contiguous CUDA tensor of 64-bit counters is required")
    check(load().vpipg_zero_counts(C.c_void_p(counts.data_ptr()), counts.numel(),
                                   _stream_ptr(stream)), "vpipg_zero_counts")


def fill_uniform_points(seed: int, first: int, xs, ys, box, stream=None) -> None:
    """Counter-based device point stream (vpipg_fill_uniform_points)."""
    import torch
    dtype = F32 if xs.dtype == torch.float32 else F64
    check(load().vpipg_fill_uniform_points(seed, first, xs.numel(), *map(float, box), dtype,
                                           C.c_void_p(xs.data_ptr()), C.c_void_p(ys.data_ptr()),
                                           _stream_ptr(stream)), "fill_uniform_points")


def mix_seed(seed: int, salt: int) -> int:
    return load().vpipg_mix_seed(seed, salt)


def regular_polygon(n: int, r: float = 1.0, center=(0.0, 0.0)):
    vx, vy = np.zeros(n), np.zeros(n)
    check(load().vpipg_regular_polygon(n, r, center[0], center[1], _dptr(vx), _dptr(vy)))
    return vx, vy


def random_convex_polygon(n: int, seed: int, r: float = 1.0, center=(0.0, 0.0)):
    vx, vy = np.zeros(n), np.zeros(n)
    check(load().vpipg_random_convex_polygon(n, seed, r, center[0], center[1], _dptr(vx),
                                             _dptr(vy)))
    return vx, vy


def sample_points(count: int, box, seed: int):
    xs, ys = np.zeros(count), np.zeros(count)
    check(load().vpipg_sample_points(count, *map(float, box), seed, _dptr(xs), _dptr(ys)))
    return xs, ys
