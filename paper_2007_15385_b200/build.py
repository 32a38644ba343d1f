"""Build recipe for libvpipg.so (CUDA kernels for sm_100a + C-ABI + vpip:: C++ API).

Compiles in-tree so the shared library travels with the repository snapshot
to the GPU box. `python -m paper_2007_15385_b200.build` or
`__graft_entry__.build()`.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = PKG / "build"
LIB = PKG / "lib" / "libvpipg.so"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))
NVCC = str(CUDA_HOME / "bin" / "nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++20", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-ffp-contract=off", "-Xptxas", "-warn-spills", "-diag-suppress", "177",
    f"-I{ROOT / 'include'}", f"-I{CSRC}",
]
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off", "-Wall",
             f"-I{ROOT / 'include'}", f"-I{CSRC}", f"-I{CUDA_HOME / 'include'}"]

CU_SOURCES = ["prep.cu", "test_f32.cu", "tri_small.cu", "tri_small_hi.cu", "test_f64.cu", "fill.cu", "csr.cu", "validate.cu", "capi.cu",
              "hostpipe.cu"]
CXX_SOURCES = ["vpip_api.cpp", "comm.cpp"]


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _headers() -> list[Path]:
    return list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list((ROOT / "include").rglob("*.h*"))


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} ... {cmd[-1]}")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)


def build_variant(tag: str, defines: list[str], sources: tuple[str, ...] = ("test_f32.cu",)) -> Path:
    """Experimental kernel variant (e.g. -DVPIPG_SLAB_P=20) as lib/variants/libvpipg_<tag>.so:
    `sources` are recompiled with `defines`, everything else is the default build."""
    out = PKG / "lib" / "variants" / f"libvpipg_{tag}.so"
    vdir = OBJ / f"v_{tag}"
    vdir.mkdir(parents=True, exist_ok=True)
    out.parent.mkdir(parents=True, exist_ok=True)
    build()
    objs = []
    for s in CU_SOURCES + CXX_SOURCES:
        if s in sources:
            vobj = vdir / (s + ".o")
            _run([NVCC, *NVCC_FLAGS, *defines, "-c", str(CSRC / s), "-o", str(vobj)])
            objs.append(vobj)
        else:
            objs.append(OBJ / (s + ".o"))
    _run([NVCC, *ARCH, "-shared", "-o", str(out), *map(str, objs), "-cudart", "static",
          "-Xlinker", "--no-undefined", "-lrt", "-lpthread", "-ldl"])
    shutil.rmtree(vdir, ignore_errors=True)  # keep the tree that ships to the GPU box small
    return out


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    LIB.parent.mkdir(exist_ok=True)
    hdrs = _headers()
    jobs = []
    objs = []
    for s in CU_SOURCES:
        src, obj = CSRC / s, OBJ / (s + ".o")
        objs.append(obj)
        if _stale(obj, [src] + hdrs):
            jobs.append([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)])
    for s in CXX_SOURCES:
        src, obj = CSRC / s, OBJ / (s + ".o")
        objs.append(obj)
        if _stale(obj, [src] + hdrs):
            jobs.append(["g++", *CXX_FLAGS, "-c", str(src), "-o", str(obj)])
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        for f in [ex.submit(_run, j) for j in jobs]:
            f.result()
    if jobs or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-cudart", "static",
              "-Xlinker", "--no-undefined", "-lrt", "-lpthread", "-ldl"])
    cli = PKG / "bin" / "vpipg"
    cli_src = CSRC / "cli" / "vpipg_cli.cpp"
    if _stale(cli, [cli_src, LIB] + hdrs):
        cli.parent.mkdir(exist_ok=True)
        _run(["g++", *CXX_FLAGS, str(cli_src), "-o", str(cli), f"-L{LIB.parent}", "-lvpipg",
              f"-L{CUDA_HOME / 'lib64'}", "-lcudart", "-Wl,-rpath,$ORIGIN/../lib",
              f"-Wl,-rpath,{CUDA_HOME / 'lib64'}"])
    timing = PKG / "bin" / "prepare_timing"
    timing_src = CSRC / "cli" / "prepare_timing.cpp"
    if _stale(timing, [timing_src, LIB] + hdrs):
        _run(["g++", *CXX_FLAGS, str(timing_src), "-o", str(timing), f"-L{LIB.parent}", "-lvpipg",
              f"-L{CUDA_HOME / 'lib64'}", "-lcudart", "-Wl,-rpath,$ORIGIN/../lib",
              f"-Wl,-rpath,{CUDA_HOME / 'lib64'}"])
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(verbose=True)
