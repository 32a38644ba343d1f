"""Device-side engine cross-validation (run_validation, bench.cpp:279-308) and
the full-size parity property at BASELINE.json's 2^31-point C5 config."""
import numpy as np
import pytest

from conftest import case_names
import workloads as W

torch = pytest.importorskip("torch")
import paper_2007_15385_b200 as vp  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def test_device_validation_equals_reference_run_validation(golden, orc):
    """f64 engines + band classification on the device reproduce the reference's
    ValidationReport (pair counts, disagreeing points, verdict) on every golden case."""
    for name in case_names(golden):
        pre = f"case_{name}_"
        vx, vy = golden[pre + "v"]
        rc, cvx, cvy, _ = orc.validate(vx, vy)  # run_validation uses polygon.vertices()
        assert rc == 0
        xs, ys = golden[pre + "pts"].astype(np.float64)
        want = golden[pre + "validation"]
        with vp.PreparedPolygon.prepare(cvx, cvy, vp.KIND_ALL) as p:
            rep = p.validate(torch.as_tensor(xs, device=DEV), torch.as_tensor(ys, device=DEV),
                             band=1e-9)
        assert rep["pair_disagreements"] == want[:3].tolist(), name
        assert rep["disagreeing_points"] == want[3], name
        assert rep["pass"] == bool(want[4]), name
        assert rep["point_count"] == xs.size


def test_validation_samples_and_failures():
    # a square with points exactly on and far off its boundary: the f32 crossing
    # kernel (no on-segment latch) disagrees with the others exactly on edges
    vx, vy = np.array([0., 1, 1, 0]), np.array([0., 0, 1, 1])
    xs = torch.tensor([0.5, 1.0, 0.25, 2.0, 1.0], dtype=torch.float32, device=DEV)
    ys = torch.tensor([0.5, 0.5, 0.0, 2.0, 1.0], dtype=torch.float32, device=DEV)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        rep = p.validate(xs, ys, band=1e-9)
        assert rep["pass"] and rep["outside_band"] == 0
        for i, d in zip(rep["sample_index"], rep["sample_dist"]):
            assert d <= 1e-9 and i in (1, 2, 4)
        # two different masks: disagreements far from any edge line fail the check
        w_a = torch.tensor([0b00001], dtype=torch.int32, device=DEV)
        w_b = torch.tensor([0b01000], dtype=torch.int32, device=DEV)  # point 3 (2, 2) is far outside
        rep = p.compare_masks(xs, ys, w_a, w_b, band=1e-5)
        assert not rep["pass"] and rep["outside_band"] == 2 and rep["disagreeing_points"] == 2
        assert rep["sample_index"] == [0, 3]


def test_c5_full_scale_parity():
    """BASELINE.json config 5 at full size (2^31 points):
    * the benchmarked fused three-engine kernel writes exactly the words and
      counts of the three per-engine kernels;
    * every fp32 engine equals the reference-exact fp64 engine of the same
      (f32) points outside the 1e-5 relative band;
    * the three fp32 engines agree with each other outside the band."""
    vx, vy = W.c5_polygon(vp.random_convex_polygon)
    m = W.C5_POINTS
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty(m, dtype=torch.float32, device=DEV)
    vp.fill_uniform_points(W.c5_point_seed(), 0, xs, ys, W.C5_BOX)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        assert p.multi_fused(xs, ys)
        fw = [torch.zeros(m // 32, dtype=torch.int32, device=DEV) for _ in range(3)]
        fc = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        p.test_multi(xs, ys, words=fw, counts=fc)
        for e in range(3):
            w = torch.zeros(m // 32, dtype=torch.int32, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, xs, ys, words=w, count=c)
            torch.cuda.synchronize()
            assert torch.equal(w, fw[e]), f"fused kernel words differ from engine {e}"
            assert c.item() == fc[e].item()
            del w
        del fw
        rep = p.validate(xs, ys, band=1e-5, relative=True)
        assert rep["pass"], rep
        assert rep["disagreeing_points"] < m * 1e-6
    d = _f32_vs_f64_all_engines(vx, vy, xs, ys)
    assert max(d) < m * 1e-6
    print("C5 2^31: f32/f64 band disagreements per engine", d,
          "three-engine disagreements:", rep["disagreeing_points"])


def _f32_vs_f64_all_engines(vx, vy, xs, ys):
    """Every engine: fp32 mask vs the reference-exact fp64 mask of the same
    (f32) points, classified on the device; disagreements must all lie in the
    1e-5 relative band. Returns the per-engine disagreement counts."""
    m = xs.numel()
    xd, yd = xs.double(), ys.double()
    out = []
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            w32 = torch.empty((m + 31) // 32, dtype=torch.int32, device=DEV)
            w64 = torch.empty_like(w32)
            c32 = torch.zeros(1, dtype=torch.int64, device=DEV)
            c64 = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, xs, ys, words=w32, count=c32)
            p.test(e, xd, yd, words=w64, count=c64)
            torch.cuda.synchronize()
            cmp = p.compare_masks(xd, yd, w64, w32, band=1e-5, relative=True)
            assert cmp["pass"], (e, cmp)
            assert abs(c32.item() - c64.item()) <= cmp["disagreeing_points"]
            out.append(cmp["disagreeing_points"])
    return out


@pytest.mark.parametrize("n", W.C3_NS)
def test_c3_full_scale_f32_vs_f64(n):
    """BASELINE.json config 3 at full size (2^28 points per n): every fp32 engine
    equals the reference-exact fp64 engine outside the band."""
    vx, vy = W.c3_polygon(n)
    m = W.C3_POINTS
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty(m, dtype=torch.float32, device=DEV)
    vp.fill_uniform_points(int(W.mix_seed_np(W.config_seed(3), 200 + n)), 0, xs, ys, W.C3_BOX)
    d = _f32_vs_f64_all_engines(vx, vy, xs, ys)
    assert max(d) < m * 1e-5
    print(f"C3 n={n}: f32/f64 band disagreements per engine {d}")


@pytest.mark.parametrize("n", (64, 256, 1024))
def test_c3x_exact_n_full_scale_f32_vs_f64(n):
    """The unjittered exact-n C3 supplement: all n edges live, up to
    n = 1024, so the tables exceed anything the literal C3 hulls produce."""
    n_, (vx, vy) = W.c3_named(f"c3x:{n}")
    assert n_ == n and len(vx) == n
    m = W.C3_POINTS
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty(m, dtype=torch.float32, device=DEV)
    vp.fill_uniform_points(int(W.mix_seed_np(W.config_seed(3), 200 + n)), 0, xs, ys, W.C3_BOX)
    d = _f32_vs_f64_all_engines(vx, vy, xs, ys)
    assert max(d) < m * 1e-5
    print(f"C3x n={n}: f32/f64 band disagreements per engine {d}")


def test_c2_full_scale_f32_vs_f64():
    """BASELINE.json config 2 (vehicle 12-gon, 2^24 clustered points)."""
    vx, vy = W.c2_polygon()
    px, py = W.c2_points()
    xs = torch.as_tensor(px, device=DEV)
    ys = torch.as_tensor(py, device=DEV)
    assert xs.dtype == torch.float32 and xs.numel() == W.C2_CLUSTERS * W.C2_PER_CLUSTER
    d = _f32_vs_f64_all_engines(vx, vy, xs, ys)
    print(f"C2: f32/f64 band disagreements per engine {d}")


def test_c2_full_scale_vs_reference_library():
    """C2 at full size (2^24 clustered points) against the unmodified reference
    library itself (oracle/_ref) on the same f32 points: every disagreement
    of every engine lies inside the 1e-5 relative band."""
    import bench_cpu as BC
    import oracle
    try:
        oracle.Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")
    vx, vy = W.c2_polygon()
    px, py = W.c2_points()
    m = px.size
    xs, ys = torch.as_tensor(px, device=DEV), torch.as_tensor(py, device=DEV)
    rr = BC.RefRun(vx, vy, px, py)
    ref = rr.run(packed=True)
    rr.close()
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            w = torch.zeros((m + 31) // 32, dtype=torch.int32, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, xs, ys, words=w, count=c)
            torch.cuda.synchronize()
            par = BC.parity_entry(w, ref[e]["words"], px, py, vx, vy, m, BC.EPS32)
            assert par["outside_band"] == 0, (e, par)
            assert abs(c.item() - ref[e]["inside"]) <= par["disagree"]
            print(f"C2 engine {e}: {par['disagree']} band disagreements vs the reference")


@pytest.mark.parametrize("nv", [40, 200])
def test_non_convex_crossing_full_scale_vs_reference_library(nv):
    """Ray crossing on a random star-shaped (non-convex) polygon, 2^24 f32
    points, against the unmodified reference library's
    ray_crossing_contains_batch on the same points (raw vertices, any simple
    polygon, vpip.cpp:120-128): every disagreement lies inside the band. Both
    table placements (parameter bank at 40 vertices, shared memory at 200)."""
    import bench_cpu as BC
    import oracle
    try:
        ref = oracle.Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(nv)
    ang = np.sort(rng.uniform(0, 2 * np.pi, nv))
    rad = rng.uniform(0.3, 1.0, nv)
    vx, vy = 3.0 + rad * np.cos(ang), -2.0 + rad * np.sin(ang)
    m = 1 << 24
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty(m, dtype=torch.float32, device=DEV)
    vp.fill_uniform_points(1234 + nv, 0, xs, ys, (2.0, -3.0, 4.0, -1.0))
    hx, hy = xs.cpu().numpy(), ys.cpu().numpy()
    want = ref.full_pass(vx, vy, hx, hy, BC.cores(), engines=(2,))[0]
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_CROSSING) as p:
        w = torch.zeros(m // 32, dtype=torch.int32, device=DEV)
        c = torch.zeros(1, dtype=torch.int64, device=DEV)
        p.test(2, xs, ys, words=w, count=c)
        torch.cuda.synchronize()
    par = BC.parity_entry(w, want["words"], hx, hy, vx, vy, m, BC.EPS32)
    assert par["outside_band"] == 0, par
    assert abs(c.item() - want["inside"]) <= par["disagree"]
    assert 0.1 < want["inside"] / m < 0.6
    print(f"non-convex {nv}-gon: {par['disagree']} band disagreements vs the reference")
