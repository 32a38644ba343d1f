"""ctypes binding of libvpipg.so (the C-ABI declared in include/vpipg.h).

The library is built in-tree by paper_2007_15385_b200/build.py. Loading fails
loudly when it is missing: there is no CPU fallback for any engine call.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# VPIPG_LIBRARY overrides the in-tree library (kernel-variant experiments only)
LIB_PATH = Path(os.environ.get("VPIPG_LIBRARY") or
                Path(__file__).resolve().parent / "lib" / "libvpipg.so")

ENGINE_VORONOI, ENGINE_OFFSET, ENGINE_CROSSING = 0, 1, 2
ENGINES = {"voronoi": 0, "sign_of_offset": 1, "offset": 1, "ray_crossing": 2, "crossing": 2}
ENGINE_NAMES = ("voronoi", "sign_of_offset", "ray_crossing")
KIND_VORONOI, KIND_OFFSET, KIND_CROSSING, KIND_ALL = 1, 2, 4, 7
F64, F32 = 0, 1
ERR_ARCH, ERR_NCCL_MISSING, ERR_NCCL, ERR_CUDA = 100, 101, 200, 1000

REPORT_SAMPLES = 100


class Report(C.Structure):
    """vpipg_report (include/vpipg.h): run_validation's ValidationReport (bench.hpp:84-102)."""
    _fields_ = [("point_count", C.c_uint64), ("pair_disagreements", C.c_uint64 * 3),
                ("disagreeing_points", C.c_uint64), ("outside_band", C.c_uint64),
                ("pass_", C.c_int), ("n_samples", C.c_uint32),
                ("sample_index", C.c_uint64 * REPORT_SAMPLES),
                ("sample_dist", C.c_double * REPORT_SAMPLES),
                ("sample_engines", C.c_uint32 * REPORT_SAMPLES)]


# name -> (restype, argtypes); every symbol include/vpipg.h declares.
_P = C.c_void_p
_D = C.POINTER(C.c_double)
SIGNATURES = {
    "vpipg_strerror": (C.c_char_p, [C.c_int]),
    "vpipg_abi_version": (C.c_int, []),
    "vpipg_prepare": (C.c_int, [_D, _D, C.c_uint32, C.c_uint32, C.c_int, _P, C.POINTER(_P)]),
    "vpipg_prepare_generators": (C.c_int, [_D, _D, C.c_uint32, C.c_int, _P, C.POINTER(_P)]),
    "vpipg_destroy": (None, [_P]),
    "vpipg_poly_info": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_int)]),
    "vpipg_poly_generators": (C.c_int, [_P, _D, _D]),
    "vpipg_poly_vertices": (C.c_int, [_P, _D, _D]),
    "vpipg_test": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, C.c_uint64, _P, _P, _P, _P]),
    "vpipg_test_host": (C.c_int, [_P, C.c_int, C.c_int, _P, _P, C.c_uint64, _P, _P,
                                  C.POINTER(C.c_uint64)]),
    "vpipg_test_host_multi": (C.c_int, [_P, C.c_uint32, C.c_int, _P, _P, C.c_uint64, _P, _P,
                                        C.POINTER(C.c_uint64)]),
    "vpipg_release_staging": (C.c_int, [C.c_int]),
    "vpipg_test_multi": (C.c_int, [_P, C.c_uint32, C.c_int, _P, _P, C.c_uint64, _P, _P, _P, _P]),
    "vpipg_test_multi_fused": (C.c_int, [_P, C.c_uint32, C.c_int, _P, _P, C.c_uint64]),
    "vpipg_test_gather_multi": (C.c_int, [_P, C.c_uint32, _P, _P, _P, C.c_uint64, _P, _P, _P, _P]),
    "vpipg_test_gather_host": (C.c_int, [_P, C.c_uint32, _P, _P, _P, C.c_uint64, _P, _P,
                                         C.POINTER(C.c_uint64)]),
    "vpipg_nccl_version": (C.c_int, [C.POINTER(C.c_int)]),
    "vpipg_comm_unique_id": (C.c_int, [C.c_char_p]),
    "vpipg_comm_init": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "vpipg_comm_init_all": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_void_p)]),
    "vpipg_comm_info": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "vpipg_allreduce_counts": (C.c_int, [_P, _P, C.c_int, _P]),
    "vpipg_zero_counts": (C.c_int, [_P, C.c_int, _P]),
    "vpipg_poly_status": (C.c_int, [_P]),
    "vpipg_allreduce_counts_group": (C.c_int, [C.c_int, _P, _P, C.c_int, _P]),
    "vpipg_comm_destroy": (C.c_int, [_P]),
    "vpipg_voronoi_work": (C.c_int, [_P, C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "vpipg_fill_uniform_points": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                            C.c_double, C.c_double, C.c_double, C.c_int, _P, _P, _P]),
    "vpipg_validate": (C.c_int, [_P, C.c_int, _P, _P, C.c_uint64, C.c_double, C.c_int, _P, _P]),
    "vpipg_compare_masks": (C.c_int, [_P, C.c_int, _P, _P, C.c_uint64, _P, _P, C.c_double, C.c_int,
                                      _P, _P]),
    "vpipg_prepare_csr": (C.c_int, [_P, _D, _D, C.c_uint32, C.c_uint32, C.c_int, _P,
                                    C.POINTER(_P), _P]),
    "vpipg_db_destroy": (None, [_P]),
    "vpipg_db_info": (C.c_int, [_P, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                C.POINTER(C.c_uint32)]),
    "vpipg_db_generators": (C.c_int, [_P, C.c_uint32, _D, _D]),
    "vpipg_test_gather": (C.c_int, [_P, C.c_int, _P, _P, _P, C.c_uint64, _P, _P, _P, _P]),
    "vpipg_fill_join_pairs": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32, _P, _P,
                                        _P, _P, _P, _P, _P]),
    "vpipg_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "vpipg_regular_polygon": (C.c_int, [C.c_uint32, C.c_double, C.c_double, C.c_double, _D, _D]),
    "vpipg_random_convex_polygon": (C.c_int, [C.c_uint32, C.c_uint64, C.c_double, C.c_double,
                                              C.c_double, _D, _D]),
    "vpipg_sample_points": (C.c_int, [C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double,
                                      C.c_uint64, _D, _D]),
}

_lib = None


def load() -> C.CDLL:
    """Load libvpipg.so (raising if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2007_15385_b200.build` "
                "(there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class VpipError(RuntimeError):
    """A non-zero C-ABI status. `code` 1..7 = vpip::ErrorCode + 1 (error.hpp:23-31)."""

    NAMES = {1: "TooFewVertices", 2: "NotConvex", 3: "DegenerateEdge", 4: "NonFinite",
             5: "GeneratorCollision", 6: "InvalidParameter", 7: "ParseError"}

    def __init__(self, code: int, where: str = ""):
        self.code = code
        msg = load().vpipg_strerror(code).decode()
        super().__init__(f"{where}: {msg} (code {code})" if where else f"{msg} (code {code})")

    @property
    def name(self) -> str:
        if self.code in self.NAMES:
            return self.NAMES[self.code]
        if self.code >= ERR_CUDA:
            return "CudaError"
        if self.code >= ERR_NCCL:
            return "NcclError"
        return "NcclMissing" if self.code == ERR_NCCL_MISSING else "ArchError"


def check(rc: int, where: str = "") -> None:
    if rc != 0:
        raise VpipError(rc, where)
