"""Runs the vpip:: C++ drop-in test program (tests/cpp/test_vpip_api.cpp) on the GPU."""
import importlib.util
import subprocess
from pathlib import Path

import pytest

HERE = Path(__file__).resolve().parent


def _builder():
    spec = importlib.util.spec_from_file_location("cpp_tests", HERE / "cpp" / "__init__.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_cpp_program_builds():
    assert _builder().build_cpp_tests().exists()


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    binary = _builder().build_cpp_tests()
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
