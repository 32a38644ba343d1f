"""CPU tests of bench.py's CPU legs (bench_cpu.py): the full-pass reference
runner, the mask diff and the band classifier behind the bench line's
`parity` block, and the reference arm on the C4 and C1 configs (reduced)."""
import json
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

import bench_cpu as BC
import workloads as W

ROOT = Path(__file__).resolve().parents[1]


def _ref():
    import oracle
    try:
        return oracle.Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")


def test_diff_indices_and_parity_entry(orc):
    m = 1000
    rng = np.random.default_rng(0)
    a = rng.integers(0, 2**32, (m + 31) // 32, dtype=np.uint64).astype(np.uint32)
    a[-1] &= (1 << (m % 32)) - 1
    b = a.copy()
    flips = [3, 64, 65, 999]
    for i in flips:
        b[i >> 5] ^= np.uint32(1 << (i & 31))
    assert BC.diff_indices(a, b, m).tolist() == flips
    # a unit square; points 3 and 64 sit far from every edge line, 65 and
    # 999 within 1e-7 of one: two disagreements outside the band
    vx, vy = np.array([0.0, 1, 1, 0]), np.array([0.0, 0, 1, 1])
    xs = np.full(m, 5.0)
    ys = np.full(m, 5.0)
    xs[[3, 64]] = [0.5, 0.3]
    ys[[3, 64]] = [0.5, 0.6]
    xs[[65, 999]] = [1.0 + 1e-7, 0.5]
    ys[[65, 999]] = [0.5, 1e-8]
    assert BC.parity_entry(a, b, xs, ys, vx, vy, m, BC.EPS32) == {"disagree": 4, "outside_band": 2}
    assert BC.parity_entry(a, a, xs, ys, vx, vy, m, BC.EPS32) == {"disagree": 0, "outside_band": 0}


def test_full_pass_equals_reference_batches(orc):
    """RefRun (chunked PointBatches, packed words, timed batch calls and
    count_inside) gives the reference's own masks and counts."""
    ref = _ref()
    vx, vy, xs, ys = BC.host_workload("c5", (1 << 16) + 77)
    rr = BC.RefRun(vx, vy, xs, ys, threads=2)
    res = rr.run(packed=True)
    rr.close()
    masks, _ = ref.masks(vx, vy, xs.astype(np.float64), ys.astype(np.float64), threads=2)
    for e in range(3):
        packed = np.packbits(masks[e], bitorder="little")
        assert np.array_equal(res[e]["words"].view(np.uint8)[:packed.size], packed)
        assert res[e]["inside"] == int(masks[e].sum())
        assert res[e]["ns"] > 0 and res[e]["count_ns"] > 0


def test_host_points_match_the_oracle_stream(orc):
    xs, ys = BC.host_points_f32(W.c5_point_seed(), 50_000, W.C5_BOX, threads=3)
    ex, ey = orc.counter_points_f32(W.c5_point_seed(), 0, 50_000, W.C5_BOX)
    assert np.array_equal(xs, ex) and np.array_equal(ys, ey)


@pytest.mark.parametrize("workload", ["c4", "c1"])
def test_reference_arm_line(workload):
    _ref()
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--workload", workload, "--points", str(1 << 18), "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and "reference library" in d["cpu_baseline"]["sample"]
