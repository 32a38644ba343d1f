"""C++ API tests: test_vpip_api.cpp exercises the vpip:: drop-in (include/vpip/)
the way the reference's doctest suites exercise the reference."""
from __future__ import annotations

import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
BIN = HERE / "test_vpip_api"


def build_cpp_tests() -> Path:
    lib = ROOT / "paper_2007_15385_b200" / "lib"
    src = HERE / "test_vpip_api.cpp"
    if BIN.exists() and BIN.stat().st_mtime > max(src.stat().st_mtime,
                                                  (lib / "libvpipg.so").stat().st_mtime):
        return BIN
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-Wall",
                    f"-I{ROOT / 'include'}", str(src), "-o", str(BIN), f"-L{lib}", "-lvpipg",
                    f"-Wl,-rpath,{lib}", "-Wl,-rpath,$ORIGIN/../../paper_2007_15385_b200/lib",
                    "-pthread"], check=True)
    return BIN
