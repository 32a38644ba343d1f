"""GPU parity: the sm_100a kernels (through the C-ABI) against the oracle.

* f64 engines repeat the reference arithmetic -> bit-exact masks and counts on
  every input, boundary points included (tolerance: none).
* f32 engines -> identical to the reference on the same f32-rounded inputs for
  every point farther than EPS32 * max(1, |x|, |y|, polygon extent) from every
  edge supporting line; disagreements inside that band are counted and
  reported (north star: 1e-5 relative for fp32).
"""
import hashlib

import numpy as np
import pytest

from conftest import case_names, unpack
import workloads as W

torch = pytest.importorskip("torch")
import paper_2007_15385_b200 as vp  # noqa: E402

pytestmark = pytest.mark.gpu
EPS32 = 1e-5
DEV = "cuda:0"


def run_device(poly, engine, xs, ys, words=True, bytes_=True):
    xs_t = torch.as_tensor(np.ascontiguousarray(xs)).to(DEV)
    ys_t = torch.as_tensor(np.ascontiguousarray(ys)).to(DEV)
    m = xs_t.numel()
    w = torch.zeros((m + 31) // 32, dtype=torch.int32, device=DEV) if words else None
    b = torch.zeros(m, dtype=torch.uint8, device=DEV) if bytes_ else None
    c = torch.zeros(1, dtype=torch.int64, device=DEV)
    poly.test(engine, xs_t, ys_t, words=w, bytes_=b, count=c)
    torch.cuda.synchronize()
    wn = w.cpu().numpy().view(np.uint32) if words else None
    bn = b.cpu().numpy() if bytes_ else None
    return wn, bn, int(c.item())


def words_to_mask(words, m):
    return np.unpackbits(words.view(np.uint8), bitorder="little")[:m]


def band_mask(orc, vx, vy, xs, ys):
    ext = max(np.ptp(vx), np.ptp(vy))
    s = np.maximum(np.maximum(1.0, np.abs(xs)), np.maximum(np.abs(ys), ext))
    return orc.edge_line_distances(np.asarray(vx, float), np.asarray(vy, float), xs, ys) <= EPS32 * s


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert torch.cuda.get_device_capability(0) == (10, 0)


def test_generators_bit_exact(golden):
    for name in golden["conv_names"]:
        vx, vy = golden[f"conv_{name}_v"]
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_VORONOI) as p:
            inner, outer = p.generators()
        assert np.array_equal(inner, golden[f"conv_{name}_inner"]), name
        assert np.array_equal(outer, golden[f"conv_{name}_outer"]), name


@pytest.mark.parametrize("name", ["too_few", "nonfinite", "degenerate", "collinear", "reflex",
                                  "pentagram", "clockwise_square"])
def test_validation_error_codes(golden, name):
    vx, vy = golden[f"val_{name}_in"]
    code = int(golden[f"val_{name}_code"])
    if code:
        with pytest.raises(vp.VpipError) as e:
            vp.PreparedPolygon.prepare(vx, vy, vp.KIND_VORONOI | vp.KIND_OFFSET)
        assert e.value.code == code
    else:
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
            ox, oy = p.vertices()
            assert p.info()[2] == bool(golden[f"val_{name}_rev"])
        assert np.array_equal(np.array([ox, oy]), golden[f"val_{name}_out"])


def test_f64_engines_bit_exact_on_all_golden_cases(golden):
    for name in case_names(golden):
        pre = f"case_{name}_"
        vx, vy = golden[pre + "v"]
        xs, ys = golden[pre + "pts"].astype(np.float64)
        want = [unpack(b, xs.size) for b in golden[pre + "masks"]]
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
            for e in range(3):
                w, b, c = run_device(p, e, xs, ys)
                assert np.array_equal(b, want[e]), (name, e, np.flatnonzero(b != want[e])[:10])
                assert np.array_equal(words_to_mask(w, xs.size), want[e]), (name, e)
                assert c == int(want[e].sum())


@pytest.mark.parametrize("name", ["c1", "square"])
def test_f64_non_finite_points_bit_exact(golden, name):
    """The f64 kernels repeat the reference's IEEE behaviour on inf / NaN /
    overflowing points too (Voronoi: inf <= inf is inside, NaN is outside;
    offset: NaN flags nothing, so inside). f32 kernels promise nothing there:
    such points have no finite distance to the boundary."""
    vx, vy = golden[f"nonfinite_{name}_v"]
    xs, ys = golden[f"nonfinite_{name}_pts"]
    want = golden[f"nonfinite_{name}_masks"]
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            w, b, c = run_device(p, e, xs, ys)
            assert np.array_equal(b, want[e]), (name, e, b.tolist(), want[e].tolist())
            assert c == int(want[e].sum())
        # and the fused exact kernel (one read of the points for all three engines)
        xt, yt = torch.as_tensor(xs, device=DEV), torch.as_tensor(ys, device=DEV)
        bs = [torch.zeros(xs.size, dtype=torch.uint8, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        p.test_multi(xt, yt, bytes_=bs, counts=cs)
        torch.cuda.synchronize()
        for e in range(3):
            assert np.array_equal(bs[e].cpu().numpy(), want[e]), (name, e)
            assert cs[e].item() == int(want[e].sum())


def test_f32_nan_points_follow_the_reference(golden, orc):
    """f32 kernels on the same points rounded to f32: a NaN coordinate gets the
    reference's IEEE answer for Voronoi (outside) and sign-of-offset (inside);
    ray crossing matches when qy is NaN (no edge is in range). A NaN qx with a
    finite qy makes the reference count only its descending edges -- that case
    is outside this fp32 kernel's promise, as are points with an infinite
    coordinate (an infinite distance is inside the relative band)."""
    for name in ("c1", "square"):
        vx, vy = golden[f"nonfinite_{name}_v"]
        with np.errstate(over="ignore"):  # 1e300 -> inf in f32
            xs, ys = golden[f"nonfinite_{name}_pts"].astype(np.float32)
        want = orc.masks(vx.astype(np.float32).astype(np.float64),
                         vy.astype(np.float32).astype(np.float64), xs.astype(np.float64),
                         ys.astype(np.float64))
        nan = np.isnan(xs) | np.isnan(ys)
        fin = np.isfinite(xs) & np.isfinite(ys)
        band = band_mask(orc, vx, vy, np.where(fin, xs, 0).astype(np.float64),
                         np.where(fin, ys, 0).astype(np.float64))
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
            for e in range(3):
                _, b, _ = run_device(p, e, xs, ys)
                check = (nan if e < 2 else np.isnan(ys)) | (fin & ~band)
                assert np.array_equal(b[check], want[e][check]), (name, e, b.tolist(), want[e].tolist())


def test_f32_engines_match_outside_band(golden, orc):
    total = {0: 0, 1: 0, 2: 0}
    for name in case_names(golden):
        pre = f"case_{name}_"
        vx, vy = golden[pre + "v"]
        xs64, ys64 = golden[pre + "pts"].astype(np.float64)
        xs, ys = xs64.astype(np.float32), ys64.astype(np.float32)
        if not bool(golden[pre + "f32"]):  # compare against the oracle on the rounded points
            want = orc.masks(vx, vy, xs.astype(np.float64), ys.astype(np.float64))
        else:
            want = [unpack(b, xs.size) for b in golden[pre + "masks"]]
        band = band_mask(orc, vx, vy, xs.astype(np.float64), ys.astype(np.float64))
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
            for e in range(3):
                w, b, c = run_device(p, e, xs, ys)
                assert np.array_equal(words_to_mask(w, xs.size), b)
                assert c == int(b.sum())
                diff = b != want[e]
                assert not np.any(diff & ~band), (name, e, np.flatnonzero(diff & ~band)[:10])
                total[e] += int(diff.sum())
                assert abs(c - int(want[e].sum())) <= int(diff.sum())
    print("f32 band disagreements per engine:", total)


def test_unit_square_known_answers():
    # test_engines.cpp:49-71, :92-106, :128-137
    with vp.PreparedPolygon.prepare([0, 1, 1, 0], [0, 0, 1, 1], vp.KIND_ALL) as p:
        pts = np.array([[0.5, 0.5], [2, 2], [1, 0.5], [2, 0.5]])
        for e in range(3):
            _, b, _ = run_device(p, e, pts[:, 0].copy(), pts[:, 1].copy())
            assert b.tolist() == [1, 0, 1, 0]
            # vertices and edge midpoints are inside under all engines (f64 exact)
            bx = np.array([0, 0.5, 1, 1, 1, 0.5, 0, 0.0])
            by = np.array([0, 0, 0, 0.5, 1, 1, 1, 0.5])
            _, b, c = run_device(p, e, bx, by)
            assert b.tolist() == [1] * 8 and c == 8


def test_concave_arrow_crossing(golden):
    vx, vy = golden["arrow_v"]
    xs, ys = golden["arrow_pts"]
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_CROSSING) as p:
        _, b, _ = run_device(p, 2, xs.copy(), ys.copy())
    assert b.tolist() == golden["arrow_inside"].tolist()
    with pytest.raises(vp.VpipError) as e:  # not convex: voronoi / offset refuse it
        vp.PreparedPolygon.prepare(vx, vy, vp.KIND_VORONOI)
    assert e.value.code == 2


@pytest.mark.parametrize("shape", ["pentagram", "comb", "clockwise_notch"])
def test_crossing_on_non_convex_polygons(orc, shape):
    """Ray crossing takes any raw polygon (vpip.cpp:120-128): a self-intersecting
    pentagram (even-odd rule: the centre is outside), a comb with many
    concavities, and a clockwise notched polygon. f64 bit-exact against the
    oracle (boundary probes included), f32 outside the band."""
    if shape == "pentagram":
        k = np.arange(5) * 2 % 5
        vx, vy = np.cos(2 * np.pi * k / 5 + np.pi / 2), np.sin(2 * np.pi * k / 5 + np.pi / 2)
    elif shape == "comb":
        teeth = 9
        xs_top = np.repeat(np.arange(teeth + 1, dtype=float), 2)[1:-1]
        ys_top = np.tile([3.0, 1.0], teeth)[: xs_top.size]
        vx = np.concatenate([[0.0, teeth], xs_top[::-1]])
        vy = np.concatenate([[0.0, 0.0], ys_top[::-1]])
    else:
        vx = np.array([0, 0, 2, 2, 3, 3, 5, 5], float)[::-1]
        vy = np.array([0, 4, 4, 1, 1, 4, 4, 0], float)[::-1]
    rng = np.random.default_rng(11)
    x0, x1, y0, y1 = vx.min() - 1, vx.max() + 1, vy.min() - 1, vy.max() + 1
    xs = np.concatenate([rng.uniform(x0, x1, 20000), vx, (vx + np.roll(vx, 1)) / 2, [0.0]])
    ys = np.concatenate([rng.uniform(y0, y1, 20000), vy, (vy + np.roll(vy, 1)) / 2, [0.0]])
    want = orc.ray_batch(vx, vy, xs, ys)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_CROSSING) as p:
        _, b, c = run_device(p, 2, xs, ys)
        assert np.array_equal(b, want) and c == int(want.sum())
        x32, y32 = xs.astype(np.float32), ys.astype(np.float32)
        want32 = orc.ray_batch(vx.astype(np.float32).astype(np.float64),
                               vy.astype(np.float32).astype(np.float64),
                               x32.astype(np.float64), y32.astype(np.float64))
        _, b32, _ = run_device(p, 2, x32, y32)
        band = band_mask(orc, vx, vy, x32.astype(np.float64), y32.astype(np.float64))
        assert not np.any((b32 != want32) & ~band)
    if shape == "pentagram":
        assert want[-1] == 0  # the centre of a pentagram is outside under even-odd


@pytest.mark.parametrize("m", [0, 1, 31, 32, 33, 255, 256, 257, 1000, 2049, 4097])
def test_ragged_sizes(orc, m):
    vx, vy = W.c1_polygon()
    xs, ys = orc.sample_points(max(m, 1), W.C1_BOX, 77 + m)
    xs, ys = xs[:m], ys[:m]
    want = orc.masks(vx, vy, xs, ys) if m else [np.zeros(0, np.uint8)] * 3
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            w, b, c = run_device(p, e, xs, ys)
            assert np.array_equal(b, want[e]) and c == int(want[e].sum())
            assert w.size == (m + 31) // 32
            assert np.array_equal(words_to_mask(w, m), want[e])
            w32, b32, c32 = run_device(p, e, xs.astype(np.float32), ys.astype(np.float32))
            assert np.array_equal(words_to_mask(w32, m), b32) and c32 == int(b32.sum())


def test_c1_full_f64_sha256(golden):
    vx, vy = W.c1_polygon()
    xs, ys = W.c1_points(vp.sample_points)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            w, _, c = run_device(p, e, xs, ys, bytes_=False)
            digest = hashlib.sha256(w.tobytes()[: (xs.size + 7) // 8]).hexdigest()
            assert digest == str(golden["c1_full_sha256"][e]), e
            assert c == int(golden["c1_full_counts"][e])


def test_device_point_stream_matches_oracle(orc):
    m, first = 100_003, 123_456_789
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty(m, dtype=torch.float32, device=DEV)
    vp.fill_uniform_points(W.c5_point_seed(), first, xs, ys, W.C5_BOX)
    ex, ey = orc.counter_points_f32(W.c5_point_seed(), first, m, W.C5_BOX)
    assert np.array_equal(xs.cpu().numpy(), ex) and np.array_equal(ys.cpu().numpy(), ey)


def test_large_batch_properties_and_shard_independence(orc):
    """2^26 f32 points (C5 polygon): masks do not depend on the partitioning
    (test_engines.cpp:227-241), popcount(words) == fused count, the three
    engines agree up to band points, and a sampled subset matches the oracle."""
    vx, vy = W.c5_polygon(vp.random_convex_polygon)
    m = 1 << 26
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty(m, dtype=torch.float32, device=DEV)
    vp.fill_uniform_points(W.c5_point_seed(), 0, xs, ys, W.C5_BOX)
    counts = []
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        full = []
        for e in range(3):
            w = torch.zeros(m // 32, dtype=torch.int32, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, xs, ys, words=w, count=c)
            # the same batch as 4 uneven 32-aligned shards
            ws = torch.zeros_like(w)
            cs = torch.zeros(1, dtype=torch.int64, device=DEV)
            cuts = [0, 32 * 1001, 32 * 777777, m - 32 * 5, m]
            for lo, hi in zip(cuts[:-1], cuts[1:]):
                p.test(e, xs[lo:hi], ys[lo:hi], words=ws[lo // 32: hi // 32], count=cs)
            torch.cuda.synchronize()
            assert torch.equal(w, ws) and c.item() == cs.item()
            pop = int(np.unpackbits(w.cpu().numpy().view(np.uint8)).sum())
            assert pop == c.item()
            counts.append(c.item())
            full.append(w.cpu().numpy().view(np.uint32))
    # three engines: differences only in band (checked exactly on a sample below)
    assert max(counts) - min(counts) <= m * 1e-5
    idx = np.sort(np.random.default_rng(5).choice(m, 200_000, replace=False))
    sx, sy = xs.cpu().numpy()[idx].astype(np.float64), ys.cpu().numpy()[idx].astype(np.float64)
    want = orc.masks(vx.astype(np.float32).astype(np.float64),
                     vy.astype(np.float32).astype(np.float64), sx, sy)
    band = band_mask(orc, vx, vy, sx, sy)
    for e in range(3):
        got = words_to_mask(full[e], m)[idx]
        assert not np.any((got != want[e]) & ~band), e


def test_host_buffer_path_equals_device_path(orc):
    vx, vy = W.c1_polygon()
    xs, ys = orc.sample_points(5_000_001, W.C1_BOX, 99)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            wd, bd, cd = run_device(p, e, xs, ys)
            wh, bh, ch = p.test_host(e, xs, ys, words=True, bytes_=True)
            assert np.array_equal(wd, wh) and np.array_equal(bd, bh) and cd == ch
            wh32, _, ch32 = p.test_host(e, xs.astype(np.float32), ys.astype(np.float32))
            wd32, _, cd32 = run_device(p, e, xs.astype(np.float32), ys.astype(np.float32),
                                       bytes_=False)
            assert np.array_equal(wd32, wh32) and cd32 == ch32


def test_host_multi_and_staging_reuse(orc):
    """vpipg_test_host_multi over several 16 Mi-point chunks equals the device
    path per engine; the per-device staging survives growth (f32 -> f64 ->
    bytes), release, and concurrent host callers on two handles."""
    import threading
    vx, vy = W.c1_polygon()
    m = (1 << 24) * 2 + 12345
    xs, ys = orc.sample_points(m, W.C1_BOX, 7)
    x32, y32 = xs.astype(np.float32), ys.astype(np.float32)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        ref = [run_device(p, e, x32, y32, bytes_=False) for e in range(3)]
        for _ in range(2):
            words, cnt = p.test_host_multi(x32, y32, (0, 1, 2))
            for e in range(3):
                assert np.array_equal(words[e], ref[e][0]) and cnt[e] == ref[e][2]
            vp.release_staging(0)
        # growth to f64 with byte masks, then back to a small f32 batch
        wh, bh, ch = p.test_host(2, xs[:3_000_001], ys[:3_000_001], words=True, bytes_=True)
        wd, bd, cd = run_device(p, 2, xs[:3_000_001], ys[:3_000_001])
        assert np.array_equal(wh, wd) and np.array_equal(bh, bd) and ch == cd
        out = {}

        def worker(k):
            with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as q:
                out[k] = q.test_host_multi(x32[: 1 << 22], y32[: 1 << 22], (0, 1, 2))

        ts = [threading.Thread(target=worker, args=(k,)) for k in range(3)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for k in range(3):
            for e in range(3):
                assert np.array_equal(out[k][0][e], ref[e][0][: (1 << 22) // 32])
    vp.release_staging(0)


@pytest.mark.parametrize("m", [4099, 1 << 20])
def test_unaligned_device_buffers(orc, m):
    """Point arrays at 4- and 12-byte offsets and a mask-word array that is not
    16-byte aligned take the guarded paths and give the same words and counts."""
    vx, vy = W.c1_polygon()
    xs, ys = orc.sample_points(m + 3, W.C1_BOX, 4242 + m)
    bx = torch.as_tensor(xs.astype(np.float32), device=DEV)
    by = torch.as_tensor(ys.astype(np.float32), device=DEV)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            ref_x, ref_y = bx[1:m + 1].clone(), by[3:m + 3].clone()
            wr = torch.zeros((m + 31) // 32, dtype=torch.int32, device=DEV)
            cr = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, ref_x, ref_y, words=wr, count=cr)
            wbuf = torch.zeros((m + 31) // 32 + 1, dtype=torch.int32, device=DEV)
            wu = wbuf[1:]
            cu = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, bx[1:m + 1], by[3:m + 3], words=wu, count=cu)
            torch.cuda.synchronize()
            assert torch.equal(wu, wr) and cu.item() == cr.item(), e
            assert wbuf[0].item() == 0


@pytest.mark.parametrize("n", [8, 2000])  # 2000: tables past the shared-memory budget
def test_outputs_have_no_stray_writes(n):
    """Canary words / bytes before and after every output region stay
    untouched for ragged sizes, both dtypes, all engines (no sanitizer on this
    pool: the kernels' bounds are checked by their side effects instead)."""
    vx, vy = vp.regular_polygon(n, 1.0)
    rng = np.random.default_rng(n)
    pad = 64
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for m in (1, 31, 33, 4099, 70001):
            for dt in (torch.float32, torch.float64):
                xs = torch.as_tensor(rng.uniform(-1.5, 1.5, m), dtype=dt, device=DEV)
                ys = torch.as_tensor(rng.uniform(-1.5, 1.5, m), dtype=dt, device=DEV)
                nw = (m + 31) // 32
                for e in range(3):
                    wbuf = torch.full((nw + 2 * pad,), -0x5a5a5a5b, dtype=torch.int32, device=DEV)
                    bbuf = torch.full((m + 2 * pad,), 0xA5, dtype=torch.uint8, device=DEV)
                    cbuf = torch.zeros(3, dtype=torch.int64, device=DEV)
                    p.test(e, xs, ys, words=wbuf[pad:pad + nw], bytes_=bbuf[pad:pad + m],
                           count=cbuf[1:2])
                    torch.cuda.synchronize()
                    w, b = wbuf.cpu().numpy(), bbuf.cpu().numpy()
                    assert (w[:pad] == -0x5a5a5a5b).all() and (w[pad + nw:] == -0x5a5a5a5b).all()
                    assert (b[:pad] == 0xA5).all() and (b[pad + m:] == 0xA5).all()
                    assert cbuf[0].item() == 0 and cbuf[2].item() == 0
                    got = b[pad:pad + m]
                    assert set(np.unique(got)) <= {0, 1}
                    bits = np.unpackbits(w[pad:pad + nw].view(np.uint8), bitorder="little")
                    assert np.array_equal(bits[:m], got) and not bits[m:].any()
                    assert cbuf[1].item() == int(got.sum())


def test_concurrent_streams_share_one_handle(orc):
    # test_engines.cpp:243-257: one generator set serves concurrent callers
    vx, vy = W.c1_polygon()
    xs, ys = orc.sample_points(1 << 20, W.C1_BOX, 5)
    xt = torch.as_tensor(xs.astype(np.float32), device=DEV)
    yt = torch.as_tensor(ys.astype(np.float32), device=DEV)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        ref = torch.zeros(xs.size // 32, dtype=torch.int32, device=DEV)
        p.test(0, xt, yt, words=ref)
        outs = [torch.zeros_like(ref) for _ in range(4)]
        streams = [torch.cuda.Stream() for _ in range(4)]
        torch.cuda.synchronize()
        for s, o in zip(streams, outs):
            p.test(0, xt, yt, words=o, stream=s)
        torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o, ref)


def test_generator_set_handle(golden):
    # voronoi_contains_batch(GeneratorSet, ...): handle from explicit generators
    name = "c1_sample"
    vx, vy = golden[f"case_{name}_v"]
    xs, ys = golden[f"case_{name}_pts"].astype(np.float64)
    want = unpack(golden[f"case_{name}_masks"][0], xs.size)
    inner, outer = golden["conv_c1_inner"], golden["conv_c1_outer"]
    with vp.PreparedPolygon.from_generators(inner, outer) as p:
        _, b, _ = run_device(p, 0, xs, ys)
        assert np.array_equal(b, want)
        with pytest.raises(vp.VpipError):  # offset tables were not prepared
            run_device(p, 1, xs, ys)


@pytest.mark.parametrize("n", [1024, 10000])
def test_many_edge_polygons_use_global_tables(orc, n):
    """Polygons whose edge tables exceed the shared-memory staging budget (the
    f64 ray records at n=1024 already do) read them from global memory;
    results stay exact (f64) / band-exact (f32)."""
    vx, vy = orc.regular_polygon(n, 1.0)
    xs, ys = orc.sample_points(20_000, (-1.2, -1.2, 1.2, 1.2), 31 + n)
    # add points hugging the boundary: the interesting region for many edges
    t = np.linspace(0, 2 * np.pi, 5000, endpoint=False)
    xs = np.concatenate([xs, 0.99999 * np.cos(t), 1.00001 * np.cos(t)])
    ys = np.concatenate([ys, 0.99999 * np.sin(t), 1.00001 * np.sin(t)])
    want = orc.masks(vx, vy, xs, ys)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            _, b, c = run_device(p, e, xs, ys)
            assert np.array_equal(b, want[e]), (n, e)
            _, b32, _ = run_device(p, e, xs.astype(np.float32), ys.astype(np.float32))
            want32 = orc.masks(vx, vy, xs.astype(np.float32).astype(np.float64),
                               ys.astype(np.float32).astype(np.float64))[e]
            band = band_mask(orc, vx, vy, xs.astype(np.float32).astype(np.float64),
                             ys.astype(np.float32).astype(np.float64))
            assert not np.any((b32 != want32) & ~band), (n, e)


def test_concurrent_prepare_test_destroy():
    """8 host threads each prepare their own polygons, test them on their own
    streams (device and host-buffer paths) and destroy them, concurrently: the
    blob pool, launch-config cache, staging and thread pool stay consistent
    (results equal a single-threaded run)."""
    import threading
    rng = np.random.default_rng(3)
    polys = [vp.random_convex_polygon(int(n), int(sd), 1.0)
             for n, sd in zip(rng.integers(3, 40, 16), rng.integers(0, 1 << 30, 16))]
    m = 300_001
    xs = torch.as_tensor(rng.uniform(-1.5, 1.5, m).astype(np.float32), device=DEV)
    ys = torch.as_tensor(rng.uniform(-1.5, 1.5, m).astype(np.float32), device=DEV)
    hx, hy = xs.cpu().numpy(), ys.cpu().numpy()

    def run(vx, vy, stream):
        out = []
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
            for e in range(3):
                w = torch.zeros((m + 31) // 32, dtype=torch.int32, device=DEV)
                c = torch.zeros(1, dtype=torch.int64, device=DEV)
                p.test(e, xs, ys, words=w, count=c, stream=stream)
                stream.synchronize()
                out.append((w.cpu().numpy(), c.item()))
            hw, hc = p.test_host_multi(hx, hy, (0, 1, 2))
        return out, hw, hc

    ref = [run(vx, vy, torch.cuda.current_stream()) for vx, vy in polys]
    got, errors = {}, []

    def worker(t):
        s = torch.cuda.Stream()
        try:
            for k in range(t, len(polys), 8):
                got[k] = run(*polys[k], s)
        except Exception as ex:  # surfaced below
            errors.append(ex)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for k in range(len(polys)):
        (o_ref, hw_ref, hc_ref), (o, hw, hc) = ref[k], got[k]
        for e in range(3):
            assert np.array_equal(o[e][0], o_ref[e][0]) and o[e][1] == o_ref[e][1]
            assert np.array_equal(hw[e], hw_ref[e]) and hc[e] == hc_ref[e]
            assert hc[e] == o[e][1]


@pytest.mark.parametrize("m", [5, 4099, 1 << 20, (1 << 22) + 777])
def test_fused_multi_engine_pass_equals_separate_calls(m):
    """vpipg_test_multi with all three engines on f32 points (the fused
    one-read kernel when the batch fits its plan, else one engine at a time)
    gives exactly the words, bytes and counts of three vpipg_test calls."""
    vx, vy = W.c5_polygon(vp.random_convex_polygon)
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    vp.fill_uniform_points(W.c5_point_seed(), 0, xs, ys, W.C5_BOX)
    # non-finite coordinates too (full slices and the guarded tail alike): the
    # fused kernel repeats the per-engine kernels' NaN / inf behaviour bit for bit
    bad = torch.as_tensor(np.random.default_rng(m).choice(m, min(m, 96), replace=False), device=DEV)
    xs[bad[0::4]] = float("nan")
    ys[bad[1::4]] = float("nan")
    xs[bad[2::4]] = float("inf")
    ys[bad[3::4]] = float("-inf")
    nw = (m + 31) // 32
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        ref = []
        for e in range(3):
            w = torch.zeros(nw, dtype=torch.int32, device=DEV)
            b = torch.zeros(m, dtype=torch.uint8, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, xs, ys, words=w, bytes_=b, count=c)
            ref.append((w, b, c))
        ws = [torch.zeros(nw, dtype=torch.int32, device=DEV) for _ in range(3)]
        bs = [torch.zeros(m, dtype=torch.uint8, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        p.test_multi(xs, ys, (0, 1, 2), words=ws, bytes_=bs, counts=cs)
        torch.cuda.synchronize()
        for e in range(3):
            assert torch.equal(ws[e], ref[e][0]) and torch.equal(bs[e], ref[e][1]), e
            assert cs[e].item() == ref[e][2].item(), e
        # the reference's IEEE answers on NaN coordinates (engines.cpp:85-98, :147-157,
        # :176-199): Voronoi outside, sign-of-offset inside, crossing outside when qy is NaN
        nan = torch.isnan(xs) | torch.isnan(ys)
        assert nan.any() and not bs[0][nan].any() and bs[1][nan].all()
        assert not bs[2][torch.isnan(ys)].any()


def _offset_table_mode(vx, vy, steep=16):
    """Python mirror of prep.cu slab_scatter's choice for the sign-of-offset
    table of a CCW polygon: 1 = y-only, 2 = x-only, 0 = two sections."""
    vx, vy = np.asarray(vx, float), np.asarray(vy, float)
    a = -(vy - np.roll(vy, 1))
    b = vx - np.roll(vx, 1)
    k = float(1 << steep)
    best, mode = None, 0
    for m, ok, lo, hi in ((1, not np.any(np.abs(a) > np.abs(b) * k), np.sum(b > 0), np.sum(b < 0)),
                          (2, not np.any(np.abs(b) > np.abs(a) * k), np.sum(a > 0), np.sum(a < 0))):
        plo, phi = max((lo + 1) & ~1, 2), max((hi + 1) & ~1, 2)
        cost = 4 * (plo + phi) + abs(plo - phi)
        if ok and (best is None or cost < best):
            best, mode = cost, m
    return mode


def _rot(vx, vy, t):
    c, s = np.cos(t), np.sin(t)
    vx, vy = np.asarray(vx, float), np.asarray(vy, float)
    return c * vx - s * vy, s * vx + c * vy


@pytest.mark.parametrize("shape", ["rect", "rect_tilted_1e-7", "one_vertical", "one_horizontal",
                                   "c5", "c2", "triangle"])
def test_slab_table_modes_match_outside_band(orc, shape):
    """The slab tables come in three forms (prep.cu): every edge a bound on y
    (one section), every edge a bound on x (one section, transposed), or the
    general two-section table when the polygon has both (near-)vertical and
    (near-)horizontal edges. Each form is held to the oracle outside the band,
    through the streaming kernels (2^20 + 13 points)."""
    if shape == "rect":
        vx, vy = [0.0, 3.0, 3.0, 0.0], [0.0, 0.0, 1.0, 1.0]
    elif shape == "rect_tilted_1e-7":
        vx, vy = _rot([0.0, 3.0, 3.0, 0.0], [0.0, 0.0, 1.0, 1.0], 1e-7)
    elif shape == "one_vertical":   # x = 2 exactly, no horizontal edge
        vx, vy = [0.0, 2.0, 2.0, -0.5], [-1.0, -0.5, 1.5, 0.7]
    elif shape == "one_horizontal":  # y = 0 exactly, no vertical edge
        vx, vy = [-1.0, 2.0, 1.3, -0.2], [0.0, 0.0, 1.7, 1.1]
    elif shape == "c5":
        vx, vy = W.c5_polygon(orc.random_convex_polygon)
    elif shape == "c2":
        vx, vy = W.c2_polygon()
    else:
        vx, vy = [0.0, 1.0, 0.3], [0.0, 0.2, 0.9]
    vx, vy = np.asarray(vx, float), np.asarray(vy, float)
    want_mode = {"rect": 0, "rect_tilted_1e-7": 0, "one_vertical": 2, "one_horizontal": 1}
    if shape in want_mode:
        assert _offset_table_mode(vx, vy) == want_mode[shape]
    m = (1 << 20) + 13
    x0, x1, y0, y1 = vx.min(), vx.max(), vy.min(), vy.max()
    pad = 0.3 * max(x1 - x0, y1 - y0)
    rng = np.random.default_rng(77)
    xs = rng.uniform(x0 - pad, x1 + pad, m).astype(np.float32)
    ys = rng.uniform(y0 - pad, y1 + pad, m).astype(np.float32)
    xs64, ys64 = xs.astype(np.float64), ys.astype(np.float64)
    want = orc.masks(vx, vy, xs64, ys64)
    band = band_mask(orc, vx, vy, xs64, ys64)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in (0, 1):
            w, b, c = run_device(p, e, xs, ys)
            assert np.array_equal(words_to_mask(w, m), b) and c == int(b.sum())
            bad = (b != want[e]) & ~band
            assert not bad.any(), (shape, e, np.flatnonzero(bad)[:5])
            assert 0.05 < b.mean() < 0.95


@pytest.mark.parametrize("shape", ["rect", "one_vertical", "one_horizontal", "triangle"])
def test_fused_pass_on_every_table_form(shape):
    """The fused kernel picks the slab table form at run time; for each form
    (two-section, x-only, y-only) its words and counts equal the separate
    single-form kernels' (2^20 + 5 points, so the fused plan applies)."""
    vx, vy = {"rect": ([0.0, 3.0, 3.0, 0.0], [0.0, 0.0, 1.0, 1.0]),
              "one_vertical": ([0.0, 2.0, 2.0, -0.5], [-1.0, -0.5, 1.5, 0.7]),
              "one_horizontal": ([-1.0, 2.0, 1.3, -0.2], [0.0, 0.0, 1.7, 1.1]),
              "triangle": ([0.0, 1.0, 0.3], [0.0, 0.2, 0.9])}[shape]
    m = (1 << 20) + 5
    rng = np.random.default_rng(5)
    xs = torch.as_tensor(rng.uniform(-1.5, 3.5, m).astype(np.float32), device=DEV)
    ys = torch.as_tensor(rng.uniform(-1.5, 2.5, m).astype(np.float32), device=DEV)
    nw = (m + 31) // 32
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        ref = []
        for e in range(3):
            w = torch.zeros(nw, dtype=torch.int32, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, xs, ys, words=w, count=c)
            ref.append((w, c))
        ws = [torch.zeros(nw, dtype=torch.int32, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        p.test_multi(xs, ys, (0, 1, 2), words=ws, counts=cs)
        torch.cuda.synchronize()
        for e in range(3):
            assert torch.equal(ws[e], ref[e][0]), (shape, e)
            assert cs[e].item() == ref[e][1].item() > 0, (shape, e)


@pytest.mark.parametrize("n", [5, 6, 7, 8, 12, 15, 16, 17, 24, 33, 40])
def test_fused_crossing_loop_forms_equal_standalone(n):
    """The fused pass runs the crossing engine's 4-edge group form for
    n <= 16 and the carried form above (test_f32.cu CrossEngine); both form
    h = qy - v.y, g = w.x - qx and d = fma(h, dvx/dvy, g) from the same
    record values, so every n mod 4 tail and both sides of the switch give
    the standalone crossing kernel's words and count bit for bit."""
    rng = np.random.default_rng(1000 + n)
    t = np.sort(rng.uniform(0.0, 2.0 * np.pi, n))
    t += np.linspace(0.0, 0.5 / n, n)  # keep the angles distinct
    vx, vy = np.cos(t), np.sin(t)
    m = (1 << 20) + 77
    xs = torch.as_tensor(rng.uniform(-1.3, 1.3, m).astype(np.float32), device=DEV)
    ys = torch.as_tensor(rng.uniform(-1.3, 1.3, m).astype(np.float32), device=DEV)
    nw = (m + 31) // 32
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        w = torch.zeros(nw, dtype=torch.int32, device=DEV)
        c = torch.zeros(1, dtype=torch.int64, device=DEV)
        p.test(2, xs, ys, words=w, count=c)
        ws = [torch.zeros(nw, dtype=torch.int32, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        p.test_multi(xs, ys, (0, 1, 2), words=ws, counts=cs)
        torch.cuda.synchronize()
        assert torch.equal(ws[2], w), n
        assert cs[2].item() == c.item() > 0, n


def test_multi_partial_engine_sets_f64_and_missing_outputs(golden):
    """vpipg_test_multi outside the fused plan: two of three engines, f64
    points, and NULL outputs for some engines -- same answers as vpipg_test,
    untouched buffers for the engines not asked for."""
    vx, vy = golden["conv_c1_v"]
    m = 70_001
    rng = np.random.default_rng(9)
    for dt in (torch.float32, torch.float64):
        xs = torch.as_tensor(rng.uniform(-1.5, 1.5, m), device=DEV).to(dt)
        ys = torch.as_tensor(rng.uniform(-1.5, 1.5, m), device=DEV).to(dt)
        nw = (m + 31) // 32
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
            ref = []
            for e in range(3):
                w = torch.zeros(nw, dtype=torch.int32, device=DEV)
                p.test(e, xs, ys, words=w)
                ref.append(w)
            ws = [torch.full((nw,), 7, dtype=torch.int32, device=DEV) for _ in range(3)]
            cs = [torch.zeros(1, dtype=torch.int64, device=DEV), None,
                  torch.zeros(1, dtype=torch.int64, device=DEV)]
            p.test_multi(xs, ys, (0, 2), words=ws, counts=cs)
            torch.cuda.synchronize()
            assert torch.equal(ws[0], ref[0]) and torch.equal(ws[2], ref[2]), dt
            assert bool((ws[1] == 7).all()), dt  # engine 1 was not requested
            for e in (0, 2):
                bits = np.unpackbits(ws[e].cpu().numpy().view(np.uint8), bitorder="little")[:m]
                assert cs[e].item() == int(bits.sum()), (dt, e)


def test_multi_fused_plan():
    """vpipg_test_multi_fused reports the route vpipg_test_multi takes: one
    fused launch for all three engines on float32 batches of polygons with at
    most 96 edges (the small-polygon kernel, route 2, for single-section
    polygons of at most 12 vertices) and on any float64 batch, per-engine
    kernels otherwise."""
    m = 1 << 20
    xs = torch.zeros(m, dtype=torch.float32, device=DEV)
    ys = torch.zeros_like(xs)
    vx, vy = W.c5_polygon(vp.random_convex_polygon)  # 32 edges
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        assert p.multi_fused(xs, ys)
        assert p.multi_route(xs, ys) == 1                 # 32 edges: the general fused kernel
        assert not p.multi_fused(xs, ys, (0, 2))
        assert p.multi_fused(xs.double(), ys.double())       # the exact f64 kernels fuse at any n
        assert not p.multi_fused(xs[:100], ys[:100])      # fewer slices than warps
        assert not p.multi_fused(xs[1:], ys[1:])          # not 16-byte aligned
    _, (vx, vy) = W.c3_named("c3:3")
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        assert p.multi_route(xs, ys) == 2                 # triangle: the small-polygon kernel
        assert p.multi_route(xs.double(), ys.double()) == 1  # f64: the exact fused kernel
        assert p.multi_route(xs[:100], ys[:100]) == 0
    _, (vx, vy) = W.c3_named("c3x:128")
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        assert not p.multi_fused(xs, ys)                  # 128 edges: separate kernels are faster
    for n, fused in ((96, True), (100, False)):           # VPIPG_FUSE_MAX_N = 96
        _, (vx, vy) = W.c3_named(f"c3x:{n}")
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
            assert p.multi_fused(xs, ys) == fused, n


@pytest.mark.parametrize("m", [7, 4099, (1 << 20) + 3])
def test_fused_f64_pass_is_reference_exact(golden, orc, m):
    """All three engines on float64 points in one fused exact kernel: masks and
    counts equal the separate exact kernels and the oracle, bit for bit."""
    vx, vy = golden["conv_c1_v"]
    xs, ys = orc.sample_points(m, W.C1_BOX, 99)
    want = orc.masks(vx, vy, xs, ys)
    xt, yt = torch.as_tensor(xs, device=DEV), torch.as_tensor(ys, device=DEV)
    nw = (m + 31) // 32
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        assert p.multi_fused(xt, yt)
        ws = [torch.zeros(nw, dtype=torch.int32, device=DEV) for _ in range(3)]
        bs = [torch.zeros(m, dtype=torch.uint8, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        p.test_multi(xt, yt, words=ws, bytes_=bs, counts=cs)
        torch.cuda.synchronize()
        for e in range(3):
            got = bs[e].cpu().numpy()
            assert np.array_equal(got, want[e]), e
            assert np.array_equal(words_to_mask(ws[e].cpu().numpy().view(np.uint32), m), got)
            assert cs[e].item() == int(want[e].sum())


@pytest.mark.parametrize("centre", [(1e3, 1e3), (-2.5e4, 7e3)])
def test_small_polygon_far_from_origin(orc, centre):
    """A unit-radius polygon far from the origin (f32 tables in the polygon's
    local frame): every engine, and the fused pass, equals the oracle outside a
    band that scales with the polygon's extent plus two f32 ulps of the
    coordinates, not with |x|."""
    cx, cy = centre
    vx, vy = vp.random_convex_polygon(24, 777, 1.0, (cx, cy))
    m = 1 << 20
    rs = np.random.default_rng(5)
    xs = (cx + rs.uniform(-1.5, 1.5, m)).astype(np.float32)
    ys = (cy + rs.uniform(-1.5, 1.5, m)).astype(np.float32)
    # plus points on and within 1e-4 of every edge line
    t = rs.uniform(0, 1, (len(vx), 64))
    ex = vx[:, None] + t * (np.roll(vx, -1)[:, None] - vx[:, None])
    ey = vy[:, None] + t * (np.roll(vy, -1)[:, None] - vy[:, None])
    xs = np.concatenate([xs, ex.ravel().astype(np.float32)])
    ys = np.concatenate([ys, (ey.ravel() + rs.uniform(-1e-4, 1e-4, ey.size)).astype(np.float32)])
    xd, yd = xs.astype(np.float64), ys.astype(np.float64)
    want = orc.masks(vx, vy, xd, yd)
    ext = max(np.ptp(vx), np.ptp(vy))
    ulp = np.spacing(np.maximum(np.abs(xs), np.abs(ys)).astype(np.float32)).astype(np.float64)
    band = orc.edge_line_distances(vx, vy, xd, yd) <= EPS32 * max(1.0, ext) + 2 * ulp
    assert band.mean() < 0.1
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for e in range(3):
            wn, bn, c = run_device(p, e, xs, ys)
            bad = (bn != want[e]) & ~band
            assert not bad.any(), (e, np.flatnonzero(bad)[:5])
        xt, yt = torch.as_tensor(xs, device=DEV), torch.as_tensor(ys, device=DEV)
        fw = [torch.zeros((xs.size + 31) // 32, dtype=torch.int32, device=DEV) for _ in range(3)]
        p.test_multi(xt, yt, words=fw)
        torch.cuda.synchronize()
        for e in range(3):
            got = words_to_mask(fw[e].cpu().numpy().view(np.uint32), xs.size)
            assert not ((got != want[e]) & ~band).any(), e


def test_python_mirror_rejects_bad_output_tensors():
    """The ctypes mirror refuses outputs the kernels would overrun: counters
    that are not 64-bit integers, mask words whose elements are not 4 bytes (or
    floats), byte masks of wider elements, too-short outputs; nothing is
    launched and no CUDA error is left behind."""
    vx, vy = np.array([0., 1, 1, 0]), np.array([0., 0, 1, 1])
    m = 100
    xs = torch.rand(m, device=DEV)
    ys = torch.rand(m, device=DEV)
    nw = (m + 31) // 32
    bad = [
        dict(count=torch.zeros(1, dtype=torch.int32, device=DEV)),
        dict(count=torch.zeros(1, dtype=torch.float64, device=DEV)),
        dict(words=torch.zeros(4 * nw, dtype=torch.uint8, device=DEV)),
        dict(words=torch.zeros(nw, dtype=torch.float32, device=DEV)),
        dict(words=torch.zeros(nw, dtype=torch.int64, device=DEV)),
        dict(words=torch.zeros(nw - 1, dtype=torch.int32, device=DEV)),
        dict(bytes_=torch.zeros(m, dtype=torch.int32, device=DEV)),
        dict(bytes_=torch.zeros(m - 1, dtype=torch.uint8, device=DEV)),
        dict(count=torch.zeros(1, dtype=torch.int64)),  # host tensor
    ]
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        for kw in bad:
            with pytest.raises(vp.VpipError) as ei:
                p.test(0, xs, ys, **kw)
            assert ei.value.code == 6, kw
            lists = {k if k != "count" else "counts": [v, None, None] for k, v in kw.items()}
            with pytest.raises(vp.VpipError):
                p.test_multi(xs, ys, **lists)
        torch.cuda.synchronize()
        w = torch.zeros(nw, dtype=torch.int32, device=DEV)
        c = torch.zeros(1, dtype=torch.int64, device=DEV)
        p.test(0, xs, ys, words=w, count=c)  # a good call still works
        torch.cuda.synchronize()
        assert c.item() == int(np.unpackbits(w.cpu().numpy().view(np.uint8)).sum())


def test_prepare_is_asynchronous_and_reports_device_status_on_first_use():
    """vpipg_prepare validates on the host (codes 1-4 at once) and only
    enqueues the device conversion: a GeneratorCollision (code 5, the
    reference's to_voronoi throw site, voronoi.cpp:46-58) surfaces at the first
    use of the handle and from vpipg_poly_status; the reference throws it for
    the same polygon."""
    # a valid but extremely thin triangle: the centroid lies within
    # 1e-12 |edge|^2 of the long edge's line
    vx, vy = np.array([0.0, 1.0, 0.5]), np.array([0.0, 0.0, 2e-12])
    with pytest.raises(vp.VpipError) as ei:  # host validation still raises at once
        vp.PreparedPolygon.prepare(np.array([0., 1, 2]), np.array([0., 0, 0]), vp.KIND_ALL)
    assert ei.value.code == 2
    p = vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL)
    assert vp.load().vpipg_poly_status(p.handle) == 5
    xs = torch.zeros(64, dtype=torch.float32, device=DEV)
    with pytest.raises(vp.VpipError) as ei:
        p.test(0, xs, xs, count=torch.zeros(1, dtype=torch.int64, device=DEV))
    assert ei.value.code == 5
    p.close()
    import oracle
    try:
        ref = oracle.Reference()
    except FileNotFoundError:
        return
    rc, _, _ = ref.to_voronoi(vx, vy)
    assert rc == 5
    # a good polygon is usable right after the (asynchronous) prepare
    q = vp.PreparedPolygon.prepare(*vp.regular_polygon(32, 1.0), vp.KIND_ALL)
    c = torch.zeros(1, dtype=torch.int64, device=DEV)
    q.test(2, xs, xs, count=c)
    torch.cuda.synchronize()
    assert c.item() == 64  # (0, 0) is inside
    q.close()


def test_first_use_of_a_fresh_handle_from_many_threads():
    """The asynchronous prepare is finished exactly once even when several host
    threads make the first call on a handle at the same time (ensure_ready),
    each on its own stream: every result equals a sequential run."""
    import threading
    vx, vy = W.c5_polygon(vp.random_convex_polygon)
    m = 1 << 20
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    vp.fill_uniform_points(99, 0, xs, ys, W.C5_BOX)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        want = []
        for e in range(3):
            w = torch.zeros(m // 32, dtype=torch.int32, device=DEV)
            p.test(e, xs, ys, words=w)
            want.append(w)
        torch.cuda.synchronize()
    for rep in range(5):
        with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:  # pending
            outs, errors = [None] * 12, []

            def worker(i):
                try:
                    s = torch.cuda.Stream()
                    with torch.cuda.stream(s):  # the zero fill ordered before the test
                        w = torch.zeros(m // 32, dtype=torch.int32, device=DEV)
                    p.test(i % 3, xs, ys, words=w, stream=s)
                    s.synchronize()
                    outs[i] = w
                except Exception as ex:
                    errors.append(ex)

            threads = [threading.Thread(target=worker, args=(i,)) for i in range(12)]
            for th in threads:
                th.start()
            for th in threads:
                th.join()
            assert not errors, errors
            for i, w in enumerate(outs):
                assert torch.equal(w, want[i % 3]), (rep, i)


@pytest.mark.parametrize("n", [3, 4, 5, 6, 7, 8, 10, 11, 12])
@pytest.mark.parametrize("form", ["y_only", "x_only", "far"])
@pytest.mark.parametrize("m", [(1 << 20) + 77, 1 << 22])
def test_small_polygon_fused_route(orc, n, form, m):
    """Polygons of at most 12 vertices whose slab tables have one section take
    the straight-line small-polygon kernel (tri_small.cu: edge count and
    padded group size compile-time, tables as constant-bank operands). Its
    words and counts equal the three per-engine kernels' bit for bit --
    y-only and x-only tables (an exactly vertical edge forces the latter),
    the local-frame shift of a polygon far from the origin, a ragged tail and
    non-finite coordinates -- and every engine equals the oracle outside the
    band."""
    rng = np.random.default_rng(4000 + 10 * n + len(form))
    t = np.sort(rng.uniform(0.0, 2.0 * np.pi, n)) + np.linspace(0.0, 0.5 / n, n)
    vx, vy = np.cos(t), np.sin(t)
    if form == "x_only":  # turn edge 0 -> 1 exactly vertical: no y-only table
        vx, vy = _rot(vx, vy, 0.5 * np.pi - np.arctan2(vy[1] - vy[0], vx[1] - vx[0]))
        vx[1] = vx[0]
    cx, cy = (300.0, -700.0) if form == "far" else (0.0, 0.0)
    vx, vy = vx + cx, vy + cy
    if form == "x_only":
        assert _offset_table_mode(vx, vy) == 2
    else:
        assert _offset_table_mode(vx, vy) != 0
    xs = (cx + rng.uniform(-1.3, 1.3, m)).astype(np.float32)
    ys = (cy + rng.uniform(-1.3, 1.3, m)).astype(np.float32)
    # non-finite coordinates past the oracle prefix: the engines' NaN / inf
    # rules must come out of the small kernel exactly as from the per-engine ones
    bad = rng.choice(np.arange(1 << 18, m), 97, replace=False)
    xs[bad[0::3]] = np.nan
    ys[bad[1::3]] = np.inf
    xs[bad[2::3]] = -np.inf
    nw = (m + 31) // 32
    xt, yt = torch.as_tensor(xs, device=DEV), torch.as_tensor(ys, device=DEV)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        assert p.multi_route(xt, yt) == 2  # the small-polygon kernel
        ref = []
        for e in range(3):
            w = torch.zeros(nw, dtype=torch.int32, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            p.test(e, xt, yt, words=w, count=c)
            ref.append((w, c))
        ws = [torch.zeros(nw, dtype=torch.int32, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        p.test_multi(xt, yt, (0, 1, 2), words=ws, counts=cs)
        torch.cuda.synchronize()
        for e in range(3):
            assert torch.equal(ws[e], ref[e][0]), (n, form, e)
            assert cs[e].item() == ref[e][1].item() > 0, (n, form, e)
    k = 1 << 18  # oracle on a prefix
    xd, yd = xs[:k].astype(np.float64), ys[:k].astype(np.float64)
    want = orc.masks(vx, vy, xd, yd)
    ext = max(np.ptp(vx), np.ptp(vy))
    ulp = np.spacing(np.maximum(np.abs(xs[:k]), np.abs(ys[:k]))).astype(np.float64)
    band = orc.edge_line_distances(vx, vy, xd, yd) <= EPS32 * max(1.0, ext) + 2 * ulp
    for e in range(3):
        got = words_to_mask(ws[e].cpu().numpy().view(np.uint32), m)[:k]
        assert not ((got != want[e]) & ~band).any(), (n, form, e)
