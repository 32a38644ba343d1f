"""Pin the CPU oracle (oracle/vpip_oracle.c) against the reference itself.

Every expected value comes from tests/golden/reference_fixtures.npz, written by
tests/golden/make_golden.py from the UNMODIFIED reference library, or from the
reference's own doctest known answers (cited inline). Bit-exact throughout.
"""
import hashlib
import math

import numpy as np
import pytest

from conftest import case_names, unpack
import workloads as W


def test_mix_seed(golden, orc):
    for (s, t), want in zip(golden["mix_seed_in"], golden["mix_seed_out"]):
        assert orc.mix_seed(int(s), int(t)) == int(want)


def test_sample_points_mt19937_64(golden, orc):
    xs, ys = orc.sample_points(1000, (-1, -1, 2, 2), 4242)
    assert np.array_equal(xs, golden["sample_xs"]) and np.array_equal(ys, golden["sample_ys"])


def test_regular_and_random_polygons(golden, orc):
    for n in range(3, 17):
        assert np.array_equal(np.stack(orc.regular_polygon(n, 1.0)), golden[f"regular_{n}"])
    for i, (n, s) in enumerate(golden["rcp_params"]):
        got = np.stack(orc.random_convex_polygon(int(n), int(s), 1.0))
        assert np.array_equal(got, golden[f"rcp_{i}"]), (n, s)


@pytest.mark.parametrize("name", ["too_few", "nonfinite", "degenerate", "collinear", "reflex",
                                  "pentagram", "clockwise_square"])
def test_validation_codes(golden, orc, name):
    vx, vy = golden[f"val_{name}_in"]
    rc, ox, oy, rev = orc.validate(vx, vy)
    assert rc == int(golden[f"val_{name}_code"])
    if rc == 0:
        assert np.array_equal(np.array([ox, oy]), golden[f"val_{name}_out"])
        assert rev == bool(golden[f"val_{name}_rev"])


def test_known_answers_conversion(orc):
    # test_voronoi.cpp:48-52 exact coefficients
    assert list(orc.edge_coefficients((0, 0), (1, 0))[1]) == [0, 1, 0]
    assert list(orc.edge_coefficients((1, 0), (1, 1))[1]) == [-1, 0, 1]
    assert list(orc.edge_coefficients((0, 1), (1, 0))[1]) == [1, 1, -1]
    assert orc.edge_coefficients((2, 3), (2, 3))[0] == 3  # DegenerateEdge
    # test_voronoi.cpp:103-118 reflections
    assert orc.reflect((0.5, 0.5), (0, 1, 0)) == (0, (0.5, -0.5))
    assert orc.reflect((0.5, 0.5), (-1, 0, 1)) == (0, (1.5, 0.5))
    assert orc.reflect((0.5, 0.5), (1, 1, -1))[0] == 5  # GeneratorCollision
    r = orc.reflect((0.2, 0.3), (1, 1, -1))[1]
    assert abs(r[0] - 0.7) <= 1e-15 and abs(r[1] - 0.8) <= 1e-15
    assert orc.foot((0.5, 0.5), (0, 1, 0)) == (0.5, 0.0)
    # test_voronoi.cpp:133-141 unit square generators, exact
    rc, inner, outer = orc.to_voronoi(np.array([0., 1, 1, 0]), np.array([0., 0, 1, 1]))
    assert rc == 0 and list(inner) == [0.5, 0.5]
    assert outer.tolist() == [[0.5, -0.5], [1.5, 0.5], [0.5, 1.5], [-0.5, 0.5]]
    # test_geometry.cpp:135-144 quad centroid (5/6, 13/12)
    cx, cy = orc.centroid(np.array([0., 2, 2, 0]), np.array([0., 0, 1, 3]))
    assert abs(cx - 5 / 6) <= 1e-12 and abs(cy - 13 / 12) <= 1e-12
    # test_voronoi.cpp:153-162 pentagon: |p_k| = 2 cos(pi/5)
    vx, vy = orc.regular_polygon(5, 1.0)
    _, _, outer = orc.to_voronoi(vx, vy)
    assert np.allclose(np.hypot(outer[:, 0], outer[:, 1]), 1.618033988749895, rtol=1e-9)


def test_conversion_bit_exact(golden, orc):
    for name in golden["conv_names"]:
        vx, vy = golden[f"conv_{name}_v"]
        rc, ov, oyv, _ = orc.validate(vx, vy)
        rc, inner, outer = orc.to_voronoi(ov, oyv)
        assert rc == 0
        assert np.array_equal(inner, golden[f"conv_{name}_inner"]), name
        assert np.array_equal(outer, golden[f"conv_{name}_outer"]), name


def test_engine_masks_bit_exact(golden, orc):
    for name in case_names(golden):
        p = f"case_{name}_"
        vx, vy = golden[p + "v"]
        xs, ys = golden[p + "pts"].astype(np.float64)
        want = np.array([unpack(b, xs.size) for b in golden[p + "masks"]])
        got = np.array(orc.masks(vx, vy, xs, ys))
        assert np.array_equal(got, want), name


@pytest.mark.parametrize("name", ["c1", "square"])
def test_non_finite_points(golden, orc, name):
    """inf / NaN / overflowing query points: the reference's IEEE answers."""
    vx, vy = golden[f"nonfinite_{name}_v"]
    xs, ys = golden[f"nonfinite_{name}_pts"]
    got = orc.masks(vx, vy, xs, ys)
    for e in range(3):
        assert np.array_equal(got[e], golden[f"nonfinite_{name}_masks"][e]), (name, e)


def test_arrow_concave(golden, orc):
    vx, vy = golden["arrow_v"]
    for (x, y), ins, cnt in zip(golden["arrow_pts"].T, golden["arrow_inside"], golden["arrow_count"]):
        assert orc.L.vo_ray_contains(orc_d(vx), orc_d(vy), 5, x, y) == ins
        assert orc.L.vo_ray_count(orc_d(vx), orc_d(vy), 5, x, y) == cnt
    # test_engines.cpp:73-81
    assert orc.L.vo_ray_count(orc_d(vx), orc_d(vy), 5, 2.0, 2.0) == 2


def orc_d(a):
    import oracle
    return np.ascontiguousarray(a, np.float64).ctypes.data_as(oracle._D)


def test_c1_full_size(golden, orc):
    vx, vy = W.c1_polygon()
    xs, ys = W.c1_points(orc.sample_points)
    assert np.array_equal(np.array([xs[:8], ys[:8]]), golden["c1_first_xy"])
    masks = orc.masks(vx, vy, xs, ys)
    assert [int(m.sum()) for m in masks] == golden["c1_full_counts"].tolist()
    for m, h in zip(masks, golden["c1_full_sha256"]):
        assert hashlib.sha256(np.packbits(m, bitorder="little").tobytes()).hexdigest() == str(h)


def test_pack_lsb_first(orc):
    # test_io.cpp:111-121: {1,0,1,1,0,0,0,0,1} -> 0x0d, 0x01
    assert orc.pack([1, 0, 1, 1, 0, 0, 0, 0, 1]).tolist() == [0x0D, 0x01]


def test_scalar_equals_batch(golden, orc):
    # acceptance.cpp:259-278: scalar early-exit tests equal the batch masks
    import oracle
    for name in ("te3", "c1_sample", "acc_8_1"):
        p = f"case_{name}_"
        vx, vy = golden[p + "v"]
        xs, ys = golden[p + "pts"].astype(np.float64)
        mv, mo, mr = orc.masks(vx, vy, xs, ys)
        rc, cvx, cvy, _ = orc.validate(vx, vy)
        _, inner, outer = orc.to_voronoi(cvx, cvy)
        d = oracle._d
        for j in range(0, xs.size, 7):
            assert orc.L.vo_voronoi_contains(d(inner), d(np.ascontiguousarray(outer)), cvx.size, xs[j], ys[j]) == mv[j]
            assert orc.L.vo_offset_contains(d(cvx), d(cvy), cvx.size, xs[j], ys[j]) == mo[j]
            assert orc.L.vo_ray_contains(d(np.ascontiguousarray(vx)), d(np.ascontiguousarray(vy)), vx.size, xs[j], ys[j]) == mr[j]


def test_counter_points_match_workload_stream(orc):
    xs, ys = orc.counter_points_f32(W.c5_point_seed(), 1000, 64, W.C5_BOX)
    j = np.arange(1000, 1064, dtype=np.uint64)
    s = W.c5_point_seed()
    ex = (-1.5 + 3.0 * W.unit_np(s, 2 * j)).astype(np.float32)
    ey = (-1.5 + 3.0 * W.unit_np(s, 2 * j + 1)).astype(np.float32)
    assert np.array_equal(xs, ex) and np.array_equal(ys, ey)


def test_reference_acceptance_suite_if_present():
    """The reference's own 8-criterion acceptance suite (compiled from its sources)."""
    import subprocess
    import oracle
    if not oracle.REF_ACCEPTANCE.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    # criterion 6 is a wall-clock shape check of the CPU benchmark (monotone
    # within 10 %); on a shared host it can flake, so it gets three tries --
    # every other criterion must pass on every run
    for attempt in range(3):
        r = subprocess.run([str(oracle.REF_ACCEPTANCE)], capture_output=True, text=True, timeout=300)
        failed = [ln for ln in r.stdout.splitlines() if ln.startswith("[FAIL]")]
        assert all(ln.startswith("[FAIL] 6.") for ln in failed), r.stdout
        if r.returncode == 0:
            break
    assert r.returncode == 0, r.stdout
    assert "all 8 criteria passed" in r.stdout


def test_reference_unit_suites_on_the_reference():
    """The reference's own unit suites (unmodified test_engines / geometry /
    voronoi / sampling / bench .cpp) on oracle/mini_doctest against the
    reference library: all pass, so the harness is faithful."""
    import subprocess
    import oracle
    if not oracle.REF_UNIT.exists():
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    r = subprocess.run([str(oracle.REF_UNIT)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout
    assert "| 0 failed" in r.stdout


def test_join_oracle_matches_reference_batches(orc):
    """vo_join_masks (per-pair restatement) == the reference's per-polygon batch
    calls over id-grouped pairs (the C4 CPU baseline), bit for bit."""
    import oracle
    import paper_2007_15385_b200 as vp
    if not oracle.REF_SO.exists():
        pytest.skip("oracle/_ref not built")
    ref = oracle.Reference()
    off, vx, vy, cx, cy, r = W.c4_polygons(vp.random_convex_polygon, npoly=512)
    xs, ys, ids = orc.join_pairs_f32(W.c4_pair_seed(), 0, 50_000, cx, cy, r)
    masks, _ = ref.join(off, vx, vy, xs, ys, ids, threads=2)
    for e in range(3):
        want = orc.join_masks(off, vx, vy, e, xs.astype(np.float64), ys.astype(np.float64), ids)
        assert np.array_equal(masks[e], want), e
    assert 0.3 < masks[0].mean() < 0.8


def test_c4_workload_polygons_are_valid_and_deterministic(orc):
    import paper_2007_15385_b200 as vp
    a = W.c4_polygons(vp.random_convex_polygon, npoly=300)
    b = W.c4_polygons(orc.random_convex_polygon, npoly=300)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    off = a[0]
    n = off[1:] - off[:-1]
    assert n.min() >= 4 and n.max() <= 16
    assert (orc.csr_status(*a[:3]) == 0).all()
