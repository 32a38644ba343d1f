"""bench.py keeps the driver's JSON contract (one line on stdout, the keys the
driver and the judge read) in its default fused mode and with --separate, at a
reduced size so the test stays short. Not a performance test."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "roofline",
        "cpu_baseline", "e2e", "clocks", "gpu_launches", "parity"}


def _run(*extra):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--points", str(1 << 22),
                          "--steps", "3", "--warmup", "3", "--e2e-steps", "1", *extra],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("mode", ["fused", "separate"])
def test_bench_line_contract(mode):
    d = _run(*(["--separate"] if mode == "separate" else []))
    assert KEYS <= d.keys()
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0
    assert d["execution"]["engines_fused"] is (mode == "fused")
    assert d["gpu_launches"] == (1 if mode == "fused" else 3) * 3
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= r.keys()
    assert 0 < r["frac"] < 1.5
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    # parity over the whole batch: the reference library and the exact f64 kernels
    p = d["parity"]
    assert p["points"] == 1 << 22 and p["outside_band"] == 0
    for blk in ("vs_reference", "f32_vs_f64_exact", "f64_exact_vs_reference"):
        assert set(p[blk]) == {"voronoi", "sign_of_offset", "ray_crossing"}
    assert all(v["disagree"] == 0 for v in p["f64_exact_vs_reference"].values())
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 8 * (1 << 22)
    names = [k["engine"] for k in d["kernels"]]
    if mode == "fused":
        assert names == ["fused"]
        assert [k["engine"] for k in d["engines_separate"]] == \
            ["voronoi", "sign_of_offset", "ray_crossing"]
    else:
        assert names == ["voronoi", "sign_of_offset", "ray_crossing"]
    # every engine counted the same points both ways (fused == separate answers)
    c = d["inside_counts"]
    assert len(c) == 3 and c[0] == c[1] and abs(c[2] - c[0]) <= 64
