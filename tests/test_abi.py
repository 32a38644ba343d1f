"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/vpipg.h declares, carries sm_100a code, fails loudly without a
B200, and its host-side samplers reproduce the reference bit for bit."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2007_15385_b200 as vp
from paper_2007_15385_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "vpipg.h"


def header_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b(vpipg_\w+)\s*\(", text, re.M)))


def test_header_symbols_all_exported():
    lib = _lib.load()
    names = header_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.SIGNATURES) == names


def test_exported_dynamic_symbols_match_header():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = sorted(set(re.findall(r"\bT (vpipg_\w+)", out)))
    assert exported == header_symbols()


def test_library_contains_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out


def test_kernels_use_fma_and_3way_minmax():
    """The slab kernel's inner loop is FFMA + FMNMX3 (two edges per FMNMX3)."""
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True,
                          text=True, check=True).stdout
    blocks = [b for b in sass.split("Function :") if "SlabEngine" in b.split("\n")[0]]
    assert blocks
    for body in blocks:
        assert "FMNMX3" in body and "FFMA" in body
    # every streaming kernel loads its points directly after an L2 prefetch
    # (CCTL.E.PML2); the crossing engine's edge loop reads the parameter-bank
    # table into uniform registers (LDCU) and its FFMAs take them as operands
    heads = [(b.split("\n")[0], b) for b in sass.split("Function :")]
    ldg = [b for h, b in heads if "ldg_kernel" in h]
    assert ldg and all("CCTL.E.PML2" in b for b in ldg)
    cross = [b for h, b in heads if "ldg_kernel" in h and "CrossEngineILi20ELb1E" in h]
    assert cross and all("LDCU" in b and re.search(r"FFMA R\d+, R\d+, UR\d+, R\d+", b) for b in cross)


def test_strerror_and_version():
    lib = _lib.load()
    assert lib.vpipg_abi_version() == 2
    assert lib.vpipg_strerror(0) == b"ok"
    assert lib.vpipg_strerror(2) == b"not convex"
    assert lib.vpipg_strerror(5) == b"generator collision"
    assert b"sm_100" in lib.vpipg_strerror(100)
    assert b"nccl" in lib.vpipg_strerror(101)


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(vp.VpipError) as e:
        vp.PreparedPolygon.prepare([0, 1, 1, 0], [0, 0, 1, 1])
    assert e.value.code >= 1000  # CUDA error, never a silent CPU path


def test_invalid_arguments_rejected_before_device():
    lib = _lib.load()
    import ctypes as C
    h = C.c_void_p()
    assert lib.vpipg_prepare(None, None, 3, 0, 0, None, C.byref(h)) == 6  # kinds == 0
    assert lib.vpipg_prepare(None, None, 3, 8, 0, None, C.byref(h)) == 6  # unknown kind
    assert lib.vpipg_test(None, 0, 1, None, None, 0, None, None, None, None) == 6


def test_host_samplers_match_reference(golden):
    for (s, t), want in zip(golden["mix_seed_in"], golden["mix_seed_out"]):
        assert vp.mix_seed(int(s), int(t)) == int(want)
    xs, ys = vp.sample_points(1000, (-1, -1, 2, 2), 4242)
    assert np.array_equal(xs, golden["sample_xs"]) and np.array_equal(ys, golden["sample_ys"])
    for n in range(3, 17):
        assert np.array_equal(np.stack(vp.regular_polygon(n)), golden[f"regular_{n}"])
    for i, (n, s) in enumerate(golden["rcp_params"]):
        assert np.array_equal(np.stack(vp.random_convex_polygon(int(n), int(s))), golden[f"rcp_{i}"])


def test_sampler_errors():
    with pytest.raises(vp.VpipError) as e:
        vp.regular_polygon(2)
    assert e.value.code == 6
    with pytest.raises(vp.VpipError):
        vp.sample_points(4, (0, 0, 0, 1), 1)


def test_nccl_loads_at_run_time_without_a_gpu():
    """The count all-reduce's NCCL is dlopen'ed: version and unique id work on a
    CPU host; bad arguments are rejected before any device call."""
    import ctypes as C
    lib = _lib.load()
    v = C.c_int()
    assert lib.vpipg_nccl_version(C.byref(v)) == 0 and v.value >= 21800
    buf = C.create_string_buffer(128)
    assert lib.vpipg_comm_unique_id(buf) == 0 and any(buf.raw)
    h = C.c_void_p()
    assert lib.vpipg_comm_init(buf, 2, 2, 0, C.byref(h)) == 6  # rank out of range
    assert lib.vpipg_comm_init(None, 1, 0, 0, C.byref(h)) == 6
    assert lib.vpipg_allreduce_counts(None, None, 3, None) == 6
    assert lib.vpipg_comm_destroy(None) == 0
    assert b"nccl" in lib.vpipg_strerror(101).lower()


def test_python_mirror_rejects_bad_device_batches():
    """The ctypes mirror checks what the raw-pointer ABI cannot: CPU tensors,
    mismatched lengths / dtypes, short outputs -> InvalidParameter (code 6)."""
    import torch
    p = object.__new__(vp.PreparedPolygon)
    p._h, p.device = None, 0
    x = torch.zeros(64, dtype=torch.float32)
    with pytest.raises(vp.VpipError) as e:
        p.test(0, x, x)  # CPU tensors
    assert e.value.code == 6
    db = object.__new__(vp.PolygonDB)
    db._h, db.device = None, 0
    with pytest.raises(vp.VpipError) as e:
        db.test(0, x, x, torch.zeros(63, dtype=torch.int32))
    assert e.value.code == 6


def test_python_mirror_rejects_bad_host_batches():
    """The host-buffer calls read m elements through raw pointers: the mirror
    rejects mismatched lengths / dtypes, non-float points, short or wide
    caller word buffers, bad join ids, and CSR offsets past the vertex arrays
    (code 6) before anything reaches the C-ABI."""
    import torch
    p = object.__new__(vp.PreparedPolygon)
    p._h, p.device = None, 0
    x32, x64 = np.zeros(100, np.float32), np.zeros(100, np.float64)
    bad = [
        lambda: p.test_host(0, x32, x32[:99]),                 # short ys
        lambda: p.test_host(0, x32, x64),                      # mixed dtypes
        lambda: p.test_host(0, np.zeros(100, np.int64), np.zeros(100, np.int64)),
        lambda: p.test_host(0, np.zeros((10, 10), np.float32), np.zeros((10, 10), np.float32)),
        lambda: p.test_host(0, x64[::2], x64[::2]),            # strided
        lambda: p.test_host_multi(x32, x32, words=[np.zeros(3, np.uint32), None, None]),
        lambda: p.test_host_multi(x32, x32, words=[np.zeros(4, np.uint64), None, None]),
        lambda: p.test_host_multi(torch.zeros(100), torch.zeros(99)),
        lambda: p.test_host_multi([0.0] * 100, [0.0] * 100),
    ]
    db = object.__new__(vp.PolygonDB)
    db._h, db.device, db.npoly, db.offsets = None, 0, 2, np.array([0, 4, 9], np.uint32)
    ids = np.zeros(100, np.uint32)
    bad += [
        lambda: db.test_host(x64, x64, ids),                   # join points are f32
        lambda: db.test_host(x32, x32, ids[:50]),
        lambda: db.test_host(x32, x32, np.zeros(100, np.int64)),
        lambda: db.generators(2),                              # index out of range
        lambda: db.generators(1, 4),                           # polygon 1 has 5 vertices
        lambda: vp.PolygonDB.prepare([0, 4, 9], np.zeros(8), np.zeros(8)),
        lambda: vp.PolygonDB.prepare([0, 4], np.zeros(4), np.zeros(5)),
        lambda: vp.PolygonDB.prepare([], np.zeros(4), np.zeros(4)),
    ]
    for i, f in enumerate(bad):
        with pytest.raises(vp.VpipError) as e:
            f()
        assert e.value.code == 6, i
