"""GPU parity for the polygon-database join (BASELINE config 4).

Device CSR preparation against the oracle: per-polygon validation status,
bit-identical generators. Then the gathered test against the oracle on
f32-rounded pairs, for all three engines: masks are identical outside the
1e-5 relative band of the pair's own polygon, and the counts are fused
correctly.
"""
import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
import paper_2007_15385_b200 as vp  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"
EPS32 = 1e-5


def _db_inputs(npoly=2048):
    off, vx, vy, cx, cy, r = W.c4_polygons(vp.random_convex_polygon, npoly=npoly)
    # inject invalid / unusual polygons (the reference's error cases), CSR-appended
    extra = [
        ([0, 1], [0, 0]),                                  # too few (1)
        ([0, 1, 2, 1], [0, 0, 0, 1]),                      # collinear (2)
        ([0, 4, 4, 2, 0], [0, 0, 4, 1, 4]),                # reflex (2)
        ([0, 1, 1, 0], [0, 0, 0, 0]),                      # degenerate (3)
        ([0, 1, np.nan], [0, 0, 1]),                       # non-finite (4)
        ([500, 500, 501, 501], [500, 501, 501, 500]),      # clockwise: valid, reversed
    ]
    vx, vy = list(vx), list(vy)
    offs = list(off)
    cxl, cyl, rl = list(cx), list(cy), list(r)
    for ex, ey in extra:
        vx += list(map(float, ex))
        vy += list(map(float, ey))
        offs.append(offs[-1] + len(ex))
        cxl.append(float(np.nanmean(ex)))
        cyl.append(float(np.nanmean(ey)))
        rl.append(1.0)
    return (np.array(offs, np.uint32), np.array(vx), np.array(vy), np.array(cxl), np.array(cyl),
            np.array(rl))


def _band(off, vx, vy, xs, ys, ids):
    """Distance of each pair to its polygon's nearest edge line <= EPS32 * scale."""
    n = (off[1:] - off[:-1]).astype(np.int64)
    d = np.full(xs.size, np.inf)
    start = off[ids].astype(np.int64)
    nn = n[ids]
    ext = np.zeros(ids.size)
    for k in range(int(n.max())):
        has = k < nn
        i0 = np.where(has, start + k, 0)
        i1 = np.where(has, start + (k + 1) % np.maximum(nn, 1), 0)
        a = vy[i0] - vy[i1]
        b = vx[i1] - vx[i0]
        c = -(a * vx[i0] + b * vy[i0])
        with np.errstate(invalid="ignore", divide="ignore"):
            dk = np.abs(a * xs + b * ys + c) / np.hypot(a, b)
        d = np.where(has, np.minimum(d, np.nan_to_num(dk, nan=np.inf)), d)
        ext = np.where(has, np.maximum(ext, np.abs(vx[i0] - vx[start]) + np.abs(vy[i0] - vy[start])), ext)
    s = np.maximum(np.maximum(1.0, np.abs(xs)), np.maximum(np.abs(ys), ext))
    return d <= EPS32 * s


def test_csr_status_and_generators(orc):
    off, vx, vy, cx, cy, r = _db_inputs(512)
    want = orc.csr_status(off, vx, vy)
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        assert np.array_equal(db.status, want)
        assert want[-6:].tolist() == [1, 2, 2, 3, 4, 0]
        for i in list(range(0, 512, 37)) + [db.npoly - 1]:
            a, b = int(off[i]), int(off[i + 1])
            rc, cvx, cvy, _ = orc.validate(vx[a:b], vy[a:b])
            rc, inner, outer = orc.to_voronoi(cvx, cvy)
            gi, go = db.generators(i, b - a)
            assert np.array_equal(gi, inner) and np.array_equal(go, outer), i


def test_device_pair_stream_matches_oracle(orc):
    off, vx, vy, cx, cy, r = _db_inputs(1024)
    m, first = 100_001, 77_777
    dcx, dcy, dr = (torch.as_tensor(a, device=DEV) for a in (cx, cy, r))
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    ids = torch.empty(m, dtype=torch.int32, device=DEV)
    vp.fill_join_pairs(W.c4_pair_seed(), first, xs, ys, ids, dcx, dcy, dr)
    ex, ey, eid = orc.join_pairs_f32(W.c4_pair_seed(), first, m, cx, cy, r)
    assert np.array_equal(xs.cpu().numpy(), ex) and np.array_equal(ys.cpu().numpy(), ey)
    assert np.array_equal(ids.cpu().numpy().view(np.uint32), eid)


@pytest.mark.parametrize("m", [1, 33, 1 << 20])
def test_gather_masks_outside_band(orc, m):
    _gather_vs_oracle(orc, m, *_db_inputs(2048))


def test_c4_config_gather_vs_oracle(orc):
    """The real C4 database (65,536 polygons of 4-16 vertices, centres in
    [0,1000]^2) and 2^22 pairs of its pair stream, every engine vs the oracle."""
    _gather_vs_oracle(orc, 1 << 22, *W.c4_polygons(vp.random_convex_polygon))


def test_c4_full_scale_vs_reference_library():
    """C4 at full size (65,536 polygons, 2^28 pairs): the fused join kernel
    (the benchmarked step) against the unmodified reference library's
    per-polygon batch calls on the same f32 pairs: every disagreement lies in
    the pair's own polygon's 1e-5 relative band."""
    import bench_cpu as BC
    import oracle
    try:
        ref = oracle.Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")
    off, vx, vy, cx, cy, r = W.c4_polygons(vp.random_convex_polygon)
    m = W.C4_PAIRS
    dcx, dcy, dr = (torch.as_tensor(a, device=DEV) for a in (cx, cy, r))
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    ids = torch.empty(m, dtype=torch.int32, device=DEV)
    vp.fill_join_pairs(W.c4_pair_seed(), 0, xs, ys, ids, dcx, dcy, dr)
    hx, hy = xs.cpu().numpy(), ys.cpu().numpy()
    hid = ids.cpu().numpy().view(np.uint32)
    want, _ = ref.join(off, vx, vy, hx.astype(np.float64), hy.astype(np.float64), hid,
                       threads=BC.cores())
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        fw = [torch.zeros((m + 31) // 32, dtype=torch.int32, device=DEV) for _ in range(3)]
        fc = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        db.test_multi(xs, ys, ids, words=fw, counts=fc)
        torch.cuda.synchronize()
    for e in range(3):
        rw = np.packbits(want[e], bitorder="little").view(np.uint32)
        par = BC.parity_entry(fw[e], rw, hx, hy, vx, vy, m, BC.EPS32, join=(off, hid))
        assert par["outside_band"] == 0, (e, par)
        assert abs(fc[e].item() - int(want[e].sum())) <= par["disagree"]
        print(f"C4 engine {e}: {par['disagree']} band disagreements vs the reference")


def _gather_vs_oracle(orc, m, off, vx, vy, cx, cy, r):
    dcx, dcy, dr = (torch.as_tensor(a, device=DEV) for a in (cx, cy, r))
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    ids = torch.empty(m, dtype=torch.int32, device=DEV)
    vp.fill_join_pairs(W.c4_pair_seed(), 0, xs, ys, ids, dcx, dcy, dr)
    hx, hy = xs.cpu().numpy().astype(np.float64), ys.cpu().numpy().astype(np.float64)
    hid = ids.cpu().numpy().view(np.uint32)
    band = _band(off, vx, vy, hx, hy, hid)
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        for e in range(3):
            want = orc.join_masks(off, vx, vy, e, hx, hy, hid)
            w = torch.zeros((m + 31) // 32, dtype=torch.int32, device=DEV)
            b = torch.zeros(m, dtype=torch.uint8, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            db.test(e, xs, ys, ids, words=w, bytes_=b, count=c)
            torch.cuda.synchronize()
            got = b.cpu().numpy()
            bits = np.unpackbits(w.cpu().numpy().view(np.uint8), bitorder="little")[:m]
            assert np.array_equal(bits, got) and c.item() == int(got.sum())
            diff = got != want
            if e == 2:  # ray crossing on non-finite raw vertices is unspecified (inputs are finite)
                fin = np.array([np.isfinite(vx[a:b]).all() and np.isfinite(vy[a:b]).all()
                                for a, b in zip(off[:-1], off[1:])])
                diff &= fin[hid]
            assert not np.any(diff & ~band), (e, np.flatnonzero(diff & ~band)[:8])
            if m > 1000:
                assert 0.2 < want.mean() < 0.9  # the join is not trivially all-in / all-out


def test_gather_invalid_ids_and_polygons_are_outside(orc):
    off, vx, vy, cx, cy, r = _db_inputs(64)
    npoly = off.size - 1
    # pairs aimed at the injected polygons (invalid ones must test outside for
    # voronoi/offset), plus out-of-range ids
    ids = np.array([npoly - 6, npoly - 5, npoly - 4, npoly - 3, npoly - 2, npoly - 1, npoly,
                    npoly + 1000, 0xFFFFFFFF], dtype=np.uint32)
    xs = np.array([0.5, 1, 1, 0.5, 0.5, 500.5, 0, 0, 0], np.float32)
    ys = np.array([0, 0.5, 1, 0, 0.5, 500.5, 0, 0, 0], np.float32)
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        for e in range(3):
            b = torch.zeros(ids.size, dtype=torch.uint8, device=DEV)
            db.test(e, torch.as_tensor(xs, device=DEV), torch.as_tensor(ys, device=DEV),
                    torch.as_tensor(ids.view(np.int32), device=DEV), bytes_=b)
            got = b.cpu().numpy()
            want = orc.join_masks(off, vx, vy, e, xs.astype(np.float64), ys.astype(np.float64), ids)
            keep = np.ones(ids.size, bool)
            if e == 2:
                # crossing takes the raw vertices of every polygon; points on the
                # degenerate ones lie on an edge line (the parity band) and the
                # NaN vertex is unspecified: compare the concave arrow (interior
                # point), the square and the out-of-range ids
                keep[[0, 1, 3, 4]] = False
            assert np.array_equal(got[keep], want[keep]), (e, got, want)
            assert got[6:].tolist() == [0, 0, 0]
            assert got[5] == 1  # the clockwise square (reversed by validation) contains its centre


def test_gather_nan_points(orc):
    """NaN query coordinates in the join: Voronoi outside, sign-of-offset inside
    (the reference's IEEE answers, as in the single-polygon kernels)."""
    off, vx, vy, cx, cy, r = _db_inputs(64)
    ids = np.arange(8, dtype=np.uint32)
    nan = np.float32("nan")
    xs = np.array([nan, cx[1], nan, cx[3], nan, cx[5], cx[6], cx[7]], np.float32)
    ys = np.array([cy[0], nan, nan, cy[3], 1e9, cy[5] + 1e4, nan, cy[7]], np.float32)
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        for e in range(2):
            b = torch.zeros(ids.size, dtype=torch.uint8, device=DEV)
            db.test(e, torch.as_tensor(xs, device=DEV), torch.as_tensor(ys, device=DEV),
                    torch.as_tensor(ids.view(np.int32), device=DEV), bytes_=b)
            got = b.cpu().numpy()
            want = orc.join_masks(off, vx, vy, e, xs.astype(np.float64), ys.astype(np.float64), ids)
            assert np.array_equal(got, want), (e, got.tolist(), want.tolist())


@pytest.mark.parametrize("m", [0, 1, 33, 4099, 100003])
def test_gather_outputs_have_no_stray_writes(m):
    """Canaries around the join's word / byte outputs stay untouched; bits past
    m in the last word are zero."""
    off, vx, vy, cx, cy, r = _db_inputs(256)
    dcx, dcy, dr = (torch.as_tensor(a, device=DEV) for a in (cx, cy, r))
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    ids = torch.empty(m, dtype=torch.int32, device=DEV)
    vp.fill_join_pairs(W.c4_pair_seed(), 0, xs, ys, ids, dcx, dcy, dr)
    pad, nw = 64, (m + 31) // 32
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        for e in range(3):
            wbuf = torch.full((nw + 2 * pad,), -0x5a5a5a5b, dtype=torch.int32, device=DEV)
            bbuf = torch.full((m + 2 * pad,), 0xA5, dtype=torch.uint8, device=DEV)
            db.test(e, xs, ys, ids, words=wbuf[pad:pad + nw], bytes_=bbuf[pad:pad + m])
            torch.cuda.synchronize()
            w, b = wbuf.cpu().numpy(), bbuf.cpu().numpy()
            assert (w[:pad] == -0x5a5a5a5b).all() and (w[pad + nw:] == -0x5a5a5a5b).all()
            assert (b[:pad] == 0xA5).all() and (b[pad + m:] == 0xA5).all()
            bits = np.unpackbits(w[pad:pad + nw].view(np.uint8), bitorder="little")
            assert np.array_equal(bits[:m], b[pad:pad + m]) and not bits[m:].any()


def test_gather_host_buffers_equal_device_path(orc):
    """vpipg_test_gather_host (pageable numpy and pinned tensors, several chunks)
    equals the device gather per engine, words and counts."""
    off, vx, vy, cx, cy, r = _db_inputs(512)
    m = (1 << 21) + 4321
    dcx, dcy, dr = (torch.as_tensor(a, device=DEV) for a in (cx, cy, r))
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    ids = torch.empty(m, dtype=torch.int32, device=DEV)
    vp.fill_join_pairs(W.c4_pair_seed(), 0, xs, ys, ids, dcx, dcy, dr)
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        ref = []
        for e in range(3):
            w = torch.zeros((m + 31) // 32, dtype=torch.int32, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            db.test(e, xs, ys, ids, words=w, count=c)
            torch.cuda.synchronize()
            ref.append((w.cpu().numpy().view(np.uint32), c.item()))
        hx, hy, hid = xs.cpu().numpy(), ys.cpu().numpy(), ids.cpu().numpy()
        for args in ((hx, hy, hid), tuple(torch.from_numpy(a).pin_memory() for a in (hx, hy, hid))):
            words, cnt = db.test_host(*args, (0, 1, 2))
            for e in range(3):
                assert np.array_equal(words[e], ref[e][0]) and cnt[e] == ref[e][1], e


@pytest.mark.parametrize("m", [0, 1, 33, 4099, 1 << 20])
def test_fused_join_equals_separate_engines(m):
    """vpipg_test_gather_multi with all three engines (one fused kernel: offset
    and crossing share one walk over the vertex rows unless validation reversed
    or rejected the polygon) gives exactly the words, bytes and counts of three
    vpipg_test_gather calls -- on a database with the reference's error cases
    and a clockwise (reversed) polygon, out-of-range ids and NaN points."""
    off, vx, vy, cx, cy, r = _db_inputs(2048)
    npoly = off.size - 1
    dcx, dcy, dr = (torch.as_tensor(a, device=DEV) for a in (cx, cy, r))
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    ids = torch.empty(m, dtype=torch.int32, device=DEV)
    vp.fill_join_pairs(W.c4_pair_seed(), 0, xs, ys, ids, dcx, dcy, dr)
    if m > 64:  # aim some pairs at the injected polygons, past the table, and at NaN
        k = torch.arange(0, m, 97, device=DEV)
        ids[k] = torch.as_tensor((npoly - 6 + (np.arange(k.numel()) % 8)).astype(np.int32),
                                 device=DEV)
        xs[k[::5]] = float("nan")
    nw = (m + 31) // 32
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        ref = []
        for e in range(3):
            w = torch.zeros(nw, dtype=torch.int32, device=DEV)
            b = torch.zeros(m, dtype=torch.uint8, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            db.test(e, xs, ys, ids, words=w, bytes_=b, count=c)
            ref.append((w, b, c))
        ws = [torch.zeros(nw, dtype=torch.int32, device=DEV) for _ in range(3)]
        bs = [torch.zeros(m, dtype=torch.uint8, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        db.test_multi(xs, ys, ids, (0, 1, 2), words=ws, bytes_=bs, counts=cs)
        torch.cuda.synchronize()
        for e in range(3):
            assert torch.equal(ws[e], ref[e][0]) and torch.equal(bs[e], ref[e][1]), e
            assert cs[e].item() == ref[e][2].item(), e


def test_fused_join_on_the_c4_database(orc):
    """The real C4 database and 2^22 pairs: the fused join equals the separate
    gather kernels (which test_c4_config_gather_vs_oracle holds to the oracle)."""
    off, vx, vy, cx, cy, r = W.c4_polygons(vp.random_convex_polygon)
    m = 1 << 22
    dcx, dcy, dr = (torch.as_tensor(a, device=DEV) for a in (cx, cy, r))
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    ids = torch.empty(m, dtype=torch.int32, device=DEV)
    vp.fill_join_pairs(W.c4_pair_seed(), 12345, xs, ys, ids, dcx, dcy, dr)
    nw = (m + 31) // 32
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        ws = [torch.zeros(nw, dtype=torch.int32, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        db.test_multi(xs, ys, ids, words=ws, counts=cs)
        for e in range(3):
            w = torch.zeros(nw, dtype=torch.int32, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            db.test(e, xs, ys, ids, words=w, count=c)
            torch.cuda.synchronize()
            assert torch.equal(ws[e], w) and cs[e].item() == c.item(), e


def _sized_db(sizes, seed=7):
    """CSR database of vpip::random_convex_polygon(n_i) for the given sizes
    (vpip::regular_polygon above 100 vertices, where the reference sampler
    finds no well-spaced angle draw), centres in [0, 1000]^2 and radii in
    [0.5, 5] (the C4 pair stream's box)."""
    rng = np.random.default_rng(seed)
    sizes = np.asarray(sizes, np.int64)
    cx, cy = rng.uniform(0, 1000, sizes.size), rng.uniform(0, 1000, sizes.size)
    r = rng.uniform(0.5, 5.0, sizes.size)
    off = np.zeros(sizes.size + 1, np.uint32)
    off[1:] = np.cumsum(sizes)
    vx, vy = np.empty(int(off[-1])), np.empty(int(off[-1]))
    for k, n in enumerate(sizes):
        c = (float(cx[k]), float(cy[k]))
        vx[off[k]:off[k + 1]], vy[off[k]:off[k + 1]] = (
            vp.regular_polygon(int(n), float(r[k]), c) if n > 100 else
            vp.random_convex_polygon(int(n), 1000 + k, float(r[k]), c))
    return off, vx, vy, cx, cy, r


@pytest.mark.parametrize("layout", ["packed", "fixed_wide"])
def test_join_polygons_above_16_vertices(orc, layout):
    """Polygons whose rows run past the header's first two 4-row chunks and the
    loop's chunk pairs: a 4..16 database with a few 17..1000-gons (records
    packed with per-polygon offsets, the largest record is far above 1.5x the
    mean) and a 17..24-gon database (fixed stride). Every engine against the
    oracle outside the band, and the fused join equal to the separate kernels."""
    rng = np.random.default_rng(11)
    if layout == "packed":
        sizes = np.concatenate([rng.integers(4, 17, 1020), [17, 20, 33, 64, 100, 255, 500, 1000]])
    else:
        sizes = rng.integers(17, 25, 1024)
    off, vx, vy, cx, cy, r = _sized_db(rng.permutation(sizes))
    m = 1 << 18
    _gather_vs_oracle(orc, m, off, vx, vy, cx, cy, r)
    dcx, dcy, dr = (torch.as_tensor(a, device=DEV) for a in (cx, cy, r))
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    ids = torch.empty(m, dtype=torch.int32, device=DEV)
    vp.fill_join_pairs(W.c4_pair_seed(), 0, xs, ys, ids, dcx, dcy, dr)
    nw = (m + 31) // 32
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        assert not db.status.any()
        ws = [torch.zeros(nw, dtype=torch.int32, device=DEV) for _ in range(3)]
        cs = [torch.zeros(1, dtype=torch.int64, device=DEV) for _ in range(3)]
        db.test_multi(xs, ys, ids, words=ws, counts=cs)
        for e in range(3):
            w = torch.zeros(nw, dtype=torch.int32, device=DEV)
            c = torch.zeros(1, dtype=torch.int64, device=DEV)
            db.test(e, xs, ys, ids, words=w, count=c)
            torch.cuda.synchronize()
            assert torch.equal(ws[e], w) and cs[e].item() == c.item(), e


def test_empty_host_batches():
    """m = 0 through every host-buffer entry point: no work, zero counts, empty
    word arrays (the reference's batch calls accept an empty PointBatch)."""
    off, vx, vy, cx, cy, r = _db_inputs(64)
    e32, e64, eid = np.zeros(0, np.float32), np.zeros(0), np.zeros(0, np.uint32)
    with vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL) as db:
        words, cnt = db.test_host(e32, e32, eid)
        assert cnt == [0, 0, 0] and all(w.size == 0 for w in words)
    pvx, pvy = W.c1_polygon()
    with vp.PreparedPolygon.prepare(pvx, pvy, vp.KIND_ALL) as p:
        for e in range(3):
            w, b, c = p.test_host(e, e64, e64, words=True, bytes_=True)
            assert w.size == 0 and b.size == 0 and c == 0
        words, cnt = p.test_host_multi(e32, e32)
        assert cnt == [0, 0, 0] and all(w.size == 0 for w in words)
