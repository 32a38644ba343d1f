#!/usr/bin/env python3
"""Benchmark of the B200 point-inclusion engine (the BASELINE.json metric).

Headline workload (BASELINE.json configs[4], the config the metric "at
1/2/4/8 B200" is quoted on; it fits one GPU): one random convex 32-gon
(vpip::random_convex_polygon(32, seed, 1.0)), 2^31 float32 points uniform in
[-1.5, 1.5]^2 from the counter-based stream, sharded evenly (1024-aligned,
contiguous) over the ranks. One step = all three engines (Voronoi,
sign-of-offset, ray-crossing) over every point + one NCCL all-reduce of the
three inside counts. The three engines run as one fused kernel that reads
each point once and writes three masks and counts (vpipg_test_multi; for the
C4 join vpipg_test_gather_multi) when the library's plan takes it;
`--separate` launches the three per-engine kernels instead, and the line's
`engines_separate` always reports their times for the per-engine roofline.
value = 3 * 2^31 point-polygon tests per step / step time (max over ranks,
CUDA events). Inputs (17 GB at N=1) are far larger than L2, so no flush is
needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c5|c2|c3:<n>|c3x:<n>|c4|c1] [--separate]

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libvpip_ref.so, the unmodified reference sources; the oracle port
when that library is absent) on a bounded sample of the same workload with all
host threads, on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import workloads as W  # noqa: E402

CPU_PASSES = 3  # timed full passes of the reference in the GPU arm's cpu_baseline leg
METRIC = "point-polygon tests/sec"
UNIT = "tests/s"
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
PIPE_PEAKS_FILE = ROOT / "profiles" / "pipe_peaks_r01.json"
TRAFFIC_FILE = ROOT / "profiles" / "traffic_r02.json"
NCU_FILE = ROOT / "profiles" / "ncu_full_r02_c5.json"
# dispatch cycles per point-edge per warp lane-slot (tools/pipe_peaks.cu model:
# FFMA/FADD 1 cycle, FMNMX3/LOP3 2): slab = FFMA + FMNMX3/2, crossing =
# 1.5 FADD + FFMA + 1.5 LOP3 (paired anchoring, test_f32.cu CrossEngine)
ISSUE_CYCLES_PER_PE = {"voronoi": 2.0, "sign_of_offset": 2.0, "ray_crossing": 5.5}
# the exact f64 kernels (test_f64.cu): the reference's own operation sequence
# on the FP64 pipe (16 lanes per SMSP: every DADD / DMUL / DSETP holds it 2
# cycles): Voronoi 3 DADD + 2 DMUL + DSETP, offset 2 DMUL + DADD + DSETP,
# crossing 2 DMUL + DADD + 4 DSETP (u.y > qy, w.y > qy, on_left, lhs == rhs;
# the on-segment box only on a tie) -- the FP64-pipe bound, not counting the
# predicate / integer logic around it (ncu, profiles/ncu_full_r02_c5f64.json)
ISSUE_CYCLES_PER_PE_F64 = {"voronoi": 12.0, "sign_of_offset": 8.0, "ray_crossing": 14.0}
HBM_FALLBACK_GBS = 6650.0
# FFMA lane-ops per SM per clock on sm_100a (tools/pipe_peaks.cu: 3.79 warp-inst/clk/SM)
FFMA_PER_SM_CLK = 128


# ----------------------------------------------------------------- helpers
def env_int(name, default):
    v = os.environ.get(name)
    return int(v) if v is not None else default


def load_peaks():
    hbm, src = HBM_FALLBACK_GBS, "fallback (B200_PROFILING.md)"
    try:
        j = json.loads(PEAKS_FILE.read_text())
        hbm, src = float(j["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except Exception:
        pass
    fma = None
    try:
        for line in PIPE_PEAKS_FILE.read_text().splitlines():
            r = json.loads(line)
            if r.get("op") == "ffma_reg":
                fma = float(r["lane_ops_per_s"])
    except Exception:
        pass
    return hbm, src, fma


class ClockSampler:
    """nvidia-smi sampled during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpus: str):
        self.rows = []
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "-i", gpus,
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 8:
                self.rows.append(parts)

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.t.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons, mhz, mx, pw = set(), [], [], []
        for r in self.rows:
            try:
                mhz.append(float(r[1]))
                mx.append(float(r[2]))
                pw.append(float(r[3]))
            except ValueError:
                continue
            for nm, v in zip(names, r[4:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(mhz) if mhz else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(mhz), "reasons": sorted(reasons)}


# ----------------------------------------------------------------- workloads
def build_workload(name: str, lo: int, hi: int, torch, vp, stream):
    """Polygon vertices (f64) + this rank's device-resident f32 points."""
    dev = torch.device("cuda", torch.cuda.current_device())
    if name == "c5":
        vx, vy = W.c5_polygon(vp.random_convex_polygon)
        m = hi - lo
        xs = torch.empty(m, dtype=torch.float32, device=dev)
        ys = torch.empty(m, dtype=torch.float32, device=dev)
        vp.fill_uniform_points(W.c5_point_seed(), lo, xs, ys, W.C5_BOX, stream=stream)
    elif name.startswith("c3"):
        n, (vx, vy) = W.c3_named(name)
        m = hi - lo
        xs = torch.empty(m, dtype=torch.float32, device=dev)
        ys = torch.empty(m, dtype=torch.float32, device=dev)
        vp.fill_uniform_points(int(W.mix_seed_np(W.config_seed(3), 200 + n)), lo, xs, ys,
                               W.C3_BOX, stream=stream)
    elif name == "c2":
        vx, vy = W.c2_polygon()
        px, py = W.c2_points()
        xs = torch.as_tensor(px[lo:hi], device=dev)
        ys = torch.as_tensor(py[lo:hi], device=dev)
    elif name == "c1":
        vx, vy = W.c1_polygon()
        px, py = W.c1_points(vp.sample_points)
        xs = torch.as_tensor(px[lo:hi], device=dev)
        ys = torch.as_tensor(py[lo:hi], device=dev)
    else:
        raise SystemExit(f"unknown workload {name}")
    return vx, vy, xs, ys


def workload_size(name: str) -> int:
    return {"c5": W.C5_POINTS, "c2": W.C2_CLUSTERS * W.C2_PER_CLUSTER, "c1": W.C1_POINTS,
            "c4": W.C4_PAIRS}.get(name.split(":")[0], W.C3_POINTS)


def workload_desc(name: str) -> str:
    return {"c5": "C5 multi-GPU scaling: random convex 32-gon, 2^31 f32 points U[-1.5,1.5]^2, "
                  "3 engines + NCCL all-reduce of inside counts",
            "c2": "C2 vehicle footprint 12-gon, 2^24 f32 lidar-like clustered points",
            "c1": "C1 random 8-angle hull, 2^20 f64 points (the oracle config, exact f64 kernels)",
            "c4": "C4 polygon-database join: 65536 random convex 4..16-gons (CSR), 2^28 f32 "
                  "(point, polygon id) pairs, gathered test"}.get(
        name.split(":")[0],
        f"C3 n-sweep regular {name} " + ("unjittered exact-n" if name.startswith("c3x")
                                         else "jittered hull") + ", 2^28 f32 points")


# ----------------------------------------------------------------- CPU reference
def c4_host_pairs(sample: int | None = None):
    """The C4 database and its (point, id) pair stream on the host (oracle, bit
    for bit the device fill_join_pairs stream)."""
    import oracle
    orc = oracle.Oracle()
    off, vx, vy, cx, cy, r = W.c4_polygons(orc.random_convex_polygon)
    m = sample or W.C4_PAIRS
    xs, ys = np.empty(m, np.float32), np.empty(m, np.float32)
    ids = np.empty(m, np.uint32)
    import concurrent.futures as cf
    step = 1 << 24

    def one(lo):
        hi = min(m, lo + step)
        xs[lo:hi], ys[lo:hi], ids[lo:hi] = orc.join_pairs_f32(W.c4_pair_seed(), lo, hi - lo, cx, cy, r)

    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        list(ex.map(one, range(0, m, step)))
    return off, vx, vy, xs, ys, ids


def reference_join(off, vx, vy, xs, ys, ids, threads, packed=False):
    """C4 through the reference: one batch call per polygon over its id-grouped
    pairs (grouping untimed), polygons split over `threads` threads.
    Returns (ns per engine, packed words per engine or None)."""
    import oracle
    ref = oracle.Reference()
    masks, ns = ref.join(off, vx, vy, xs.astype(np.float64), ys.astype(np.float64), ids,
                         threads=threads)
    words = [np.packbits(mk, bitorder="little").view(np.uint8) for mk in masks] if packed else None
    if words is not None:
        words = [np.pad(w, (0, (-w.size) % 4)).view(np.uint32) for w in words]
    return ns, words, ref.build


def reference_c1(threads):
    """C1 (the f64 oracle config) through the reference: (ns per engine, byte masks)."""
    import oracle
    ref = oracle.Reference()
    vx, vy = W.c1_polygon()
    xs, ys = W.c1_points(ref.sample_points)
    masks, ns = ref.masks(vx, vy, xs, ys, threads=threads)
    return ns, masks, ref.build, (vx, vy, xs, ys)


def run_reference_arm(args, rank: int, world: int):
    """--impl reference: the reference's own CPU path on the FULL workload (the
    same config as the GPU arm), rank 0 only, all host threads; one step = one
    pass of the three engines over every point (C5: 2^31 points in 2^26-point
    PointBatch chunks), timed as run_benchmark times its batch
    calls (bench.cpp:196-199) and summed over the chunks."""
    if rank != 0:
        return
    import bench_cpu as BC
    steps, warmup, th = args.steps, args.warmup, BC.cores()
    name = args.workload
    extra = {}
    per_step = []
    if name == "c4":
        off, vx, vy, xs, ys, ids = c4_host_pairs(args.points or None)
        for r in range(warmup + steps):
            ns, _, build = reference_join(off, vx, vy, xs, ys, ids, th)
            if r >= warmup:
                per_step.append(sum(ns) * 1e-9)
        m = xs.size
        desc = (f"the unmodified reference library ({build}), all {m} pairs of the C4 stream "
                f"(f32 widened to f64), pairs grouped by polygon id (untimed), one "
                f"*_contains_batch call per polygon, polygons split over {th} threads, 3 engines")
    elif name == "c1":
        for r in range(warmup + steps):
            ns, _, build, (vx, vy, xs, ys) = reference_c1(th)
            if r >= warmup:
                per_step.append(sum(ns) * 1e-9)
        m = xs.size
        desc = (f"the unmodified reference library ({build}), all {m} f64 points of C1, 3 engines "
                f"*_contains_batch(threads={th}) timed like bench.cpp:196-199")
    else:
        vx, vy, xs, ys = BC.host_workload(name, args.points or None)
        m = xs.size
        rr = BC.RefRun(vx, vy, xs, ys, th)
        del xs, ys
        cnt = []
        for r in range(warmup + steps):
            res = rr.run()
            if r >= warmup:
                per_step.append(sum(x["ns"] for x in res) * 1e-9)
                cnt.append(sum(x["count_ns"] for x in res) * 1e-9)
        extra["count_inside_ms"] = statistics.median(cnt) * 1e3
        extra["inside_counts"] = [x["inside"] for x in res]
        desc = rr.describe()
        rr.close()
    t = statistics.median(per_step)
    value = 3 * m / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(args, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": th, "kind": "reference",
                         "sample": desc + f"; median of {steps} full passes after {warmup} "
                                          f"warm-up passes", **extra},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(args, world):
    return {"workload": workload_desc(args.workload),
            "points": args.points or workload_size(args.workload),
            "engines": ["voronoi", "sign_of_offset", "ray_crossing"],
            "parallelism": f"point shards x{world}",
            "l2": ("inputs larger than L2" if workload_size(args.workload) * 8 > 4 * 126e6
                   else "L2 flushed between steps (256 MB read, outside the step events)")}


# ----------------------------------------------------------------- GPU jobs
class PolygonJob:
    """One polygon against a device-resident point stream (C1, C2, C3, C5)."""

    issue_cycles = ISSUE_CYCLES_PER_PE
    bytes_per_unit = 8  # f32 x + y per test
    e2e_path = ("vpipg_test_host_multi (C-ABI, pinned host buffers, chunks of m/8 (1-16 Mi "
                "points) on 3 streams; one H2D per chunk feeds all 3 engines)")

    def __init__(self, workload, lo, hi, device, torch, vp, stream, dtype="f32"):
        self.torch = torch
        self.workload = workload
        vx, vy, self.xs, self.ys = build_workload(workload, lo, hi, torch, vp, stream)
        if dtype == "f64" and self.xs.dtype == torch.float32:
            # the reference's own precision: the f32 stream widened exactly, run
            # through the reference-exact f64 kernels
            self.xs, self.ys = self.xs.double(), self.ys.double()
        self.vx, self.vy = np.asarray(vx, np.float64), np.asarray(vy, np.float64)
        t0 = time.perf_counter()
        self.poly = vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL, device=device, stream=stream)
        self.prep_ms = (time.perf_counter() - t0) * 1e3
        self.n_edges = self.poly.n
        # C1 is the f64 oracle config: its points stay f64 and run the exact kernels
        self.f64 = self.xs.dtype == torch.float64
        if self.f64:
            self.bytes_per_unit = 16
            self.issue_cycles = ISSUE_CYCLES_PER_PE_F64

    def launch(self, e, words, count, stream):
        self.poly.test(e, self.xs, self.ys, words=words, count=count, stream=stream)

    def launch_all(self, words, counts, stream):
        self.poly.test_multi(self.xs, self.ys, (0, 1, 2), words=words, counts=counts, stream=stream)

    def prepare_host(self):
        t = self.torch
        self.hx = t.empty(self.xs.numel(), dtype=self.xs.dtype, pin_memory=True)
        self.hy = t.empty(self.ys.numel(), dtype=self.ys.dtype, pin_memory=True)
        self.hx.copy_(self.xs)
        self.hy.copy_(self.ys)

    def run_host(self, hw, stream):
        _, cnt = self.poly.test_host_multi(self.hx, self.hy, (0, 1, 2), words=hw)
        return cnt

    def release_host(self):
        self.hx = self.hy = None


class JoinJob:
    """C4: a CSR polygon database and (point, polygon id) pairs, gathered test."""

    # affine gather: 2 FFMA + LOP3/2 per point-edge; crossing as in the stream kernel
    issue_cycles = {"voronoi": 3.0, "sign_of_offset": 3.0, "ray_crossing": 6.0}
    bytes_per_unit = 12  # f32 x + y + u32 id per test
    e2e_path = ("vpipg_test_gather_host (C-ABI, pinned host pairs, chunks of m/8 on 3 streams; "
                "one H2D per chunk feeds all 3 engines)")

    def __init__(self, workload, lo, hi, device, torch, vp, stream, dtype="f32"):
        if dtype != "f32":
            raise SystemExit("the C4 join runs on f32 pairs")
        self.torch = torch
        off, vx, vy, cx, cy, r = W.c4_polygons(vp.random_convex_polygon)
        self.off, self.vx, self.vy = off, vx, vy
        t0 = time.perf_counter()
        self.db = vp.PolygonDB.prepare(off, vx, vy, vp.KIND_ALL, device=device, stream=stream)
        self.prep_ms = (time.perf_counter() - t0) * 1e3
        nv = (off[1:] - off[:-1]).astype(np.float64)
        self.n_edges = float(nv.mean())  # ids are uniform over the polygons
        m = hi - lo
        dev = torch.device("cuda", device)
        self.xs = torch.empty(m, dtype=torch.float32, device=dev)
        self.ys = torch.empty(m, dtype=torch.float32, device=dev)
        self.ids = torch.empty(m, dtype=torch.int32, device=dev)
        c = [torch.as_tensor(a, device=dev) for a in (cx, cy, r)]
        vp.fill_join_pairs(W.c4_pair_seed(), lo, self.xs, self.ys, self.ids, *c, stream=stream)

    def launch(self, e, words, count, stream):
        self.db.test(e, self.xs, self.ys, self.ids, words=words, count=count, stream=stream)

    def launch_all(self, words, counts, stream):
        self.db.test_multi(self.xs, self.ys, self.ids, (0, 1, 2), words=words, counts=counts,
                           stream=stream)

    def prepare_host(self):
        t = self.torch
        self.h = [t.empty(a.numel(), dtype=a.dtype, pin_memory=True) for a in (self.xs, self.ys, self.ids)]
        for hbuf, d in zip(self.h, (self.xs, self.ys, self.ids)):
            hbuf.copy_(d)

    def run_host(self, hw, stream):
        _, cnt = self.db.test_host(*self.h, (0, 1, 2), words=hw)
        return cnt

    def release_host(self):
        self.h = None


# ----------------------------------------------------------------- convert phase
def convert_block(vp, device, stream):
    """Warm preparation cost beside the reference's conversion phase
    (run_benchmark times to_voronoi, bench.cpp:165-170; validate_polygon,
    geometry.cpp:53-98, is timed separately). GPU: the C-ABI vpipg_prepare
    call (host validation + the enqueued device conversion; returns without
    waiting) and, separately, prepare + vpipg_poly_status (until the handle is
    usable), medians of 50 warm calls through ctypes; the 65,536-polygon C4
    ingest (vpipg_prepare_csr, synchronous: it returns per-polygon status),
    median of 5 warm calls."""
    import ctypes as C
    L = vp.load()
    sptr = C.c_void_p(stream.cuda_stream)
    polys = [(8, vp.random_convex_polygon(8, 11, 1.0)), (32, W.c5_polygon(vp.random_convex_polygon)),
             (1024, vp.regular_polygon(1024, 1.0))]
    try:
        import oracle
        ref = oracle.Reference()
    except Exception:
        ref = None
    # the C-ABI call's own host-visible cost, from a C++ caller (regular n-gons)
    cxx = {}
    try:
        out = subprocess.run([str(ROOT / "paper_2007_15385_b200" / "bin" / "prepare_timing"), "8",
                              "32", "1024"], capture_output=True, text=True, timeout=120,
                             env={**os.environ, "CUDA_VISIBLE_DEVICES":
                                  os.environ.get("CUDA_VISIBLE_DEVICES", str(device))})
        for line in out.stdout.splitlines():
            r = json.loads(line)
            cxx[r["n"]] = r
    except Exception:
        pass
    single = []
    for n, (vx, vy) in polys:
        vx, vy = np.ascontiguousarray(vx, np.float64), np.ascontiguousarray(vy, np.float64)
        px, py = vx.ctypes.data_as(C.POINTER(C.c_double)), vy.ctypes.data_as(C.POINTER(C.c_double))
        enq, rdy = [], []
        for r in range(60):
            h = C.c_void_p()
            t0 = time.perf_counter()
            rc = L.vpipg_prepare(px, py, n, vp.KIND_ALL, device, sptr, C.byref(h))
            t1 = time.perf_counter()
            st = L.vpipg_poly_status(h)
            t2 = time.perf_counter()
            L.vpipg_destroy(h)
            if rc or st:
                raise SystemExit(f"prepare n={n}: {rc} {st}")
            if r >= 10:
                enq.append(t1 - t0)
                rdy.append(t2 - t0)
        e = {"n": n, "prepare_enqueue_us": statistics.median(enq) * 1e6,
             "prepare_ready_us": statistics.median(rdy) * 1e6}
        if n in cxx:
            e["cxx_prepare_enqueue_us"] = cxx[n]["prepare_enqueue_us"]
            e["cxx_prepare_ready_us"] = cxx[n]["prepare_ready_us"]
        if ref is not None:
            tv, tc = ref.time_convert(vx, vy)
            e.update({"reference_validate_us": tv / 1e3, "reference_to_voronoi_us": tc / 1e3})
        single.append(e)
    ct = []
    for r in range(200):  # the ctypes call overhead included in the figures above
        t0 = time.perf_counter()
        L.vpipg_abi_version()
        ct.append(time.perf_counter() - t0)
    off, cvx, cvy, *_ = W.c4_polygons(vp.random_convex_polygon)
    ing = []
    for r in range(7):
        t0 = time.perf_counter()
        db = vp.PolygonDB.prepare(off, cvx, cvy, vp.KIND_ALL, device=device, stream=stream)
        t1 = time.perf_counter()
        db.close()
        if r >= 2:
            ing.append(t1 - t0)
    c4 = {"polygons": int(off.size - 1), "ingest_ms": statistics.median(ing) * 1e3}
    if ref is not None:
        tv, tc = ref.time_convert_csr(off, cvx, cvy)
        c4.update({"reference_validate_ms": tv / 1e6, "reference_to_voronoi_ms": tc / 1e6,
                   "reference_threads": 1})
    return {"single": single, "c4": c4, "ctypes_call_us": statistics.median(ct) * 1e6,
            "what": "warm medians; GPU: vpipg_prepare = host validate_polygon + enqueued device "
                    "conversion (generators, f32 tables), ready = until vpipg_poly_status "
                    "returns, timed through ctypes and (cxx_*) by a C++ caller "
                    "(bin/prepare_timing, regular n-gons); C4: vpipg_prepare_csr of the 65,536-polygon database. Reference: "
                    "validate_polygon and to_voronoi (the convert phase of bench.cpp:165-170) "
                    "of the same polygons, single-threaded as run_benchmark runs them"}


# ----------------------------------------------------------------- CPU leg + parity
def cpu_leg(job, words, m, torch):
    """cpu_baseline and the parity block (rank 0, N=1). The reference library
    runs the FULL workload twice on all host threads: the first pass (warm-up)
    yields its masks, the second is the timed figure. Parity compares, per
    engine, the GPU mask words of the last timed step with
      * vs_reference: the reference's masks of the same (f32-rounded) points;
      * f32_vs_f64_exact: the library's reference-exact f64 kernels over the
        whole batch (points widened on the device);
      * f64_exact_vs_reference: those f64 masks against the reference, which
        must agree bit for bit (band 1e-9);
    a disagreement counts as outside_band when the point lies farther than
    eps * max(1, |x|, |y|, polygon extent) from every edge's supporting line
    (edge_line_distance, voronoi.cpp:73-82; the C oracle's, on the host)."""
    import bench_cpu as BC
    th = BC.cores()
    names = BC.NAMES
    par = {"points": m, "band": "eps * max(1, |x|, |y|, polygon extent) from the nearest edge "
                                "supporting line (edge_line_distance, voronoi.cpp:73-82); "
                                "eps 1e-5 for f32 masks, 1e-9 for f64",
           "words": "the GPU mask words of the last timed step"}

    def block(ws_a, ws_b, xs, ys, eps, join=None):
        return {n: BC.parity_entry(ws_a[e], ws_b[e], xs, ys, job.vx, job.vy, m, eps, join)
                for e, n in enumerate(names)}

    if isinstance(job, JoinJob):
        import oracle
        xs, ys = job.xs.cpu().numpy(), job.ys.cpu().numpy()
        ids = job.ids.cpu().numpy().view(np.uint32)
        _, rw, build = reference_join(job.off, job.vx, job.vy, xs, ys, ids, th, packed=True)
        ns, _, _ = reference_join(job.off, job.vx, job.vy, xs, ys, ids, th)
        t = sum(ns) * 1e-9
        ref = oracle.Reference()
        sc = [ref.join_scalar(job.off, job.vx, job.vy, xs.astype(np.float64),
                              ys.astype(np.float64), ids, e, th)[1] for e in range(3)]
        cpu = {"value": 3 * m / t, "unit": UNIT, "cores": th, "kind": "reference",
               "sample": f"the unmodified reference library ({build}), all {m} pairs of the C4 "
                         f"stream (f32 widened to f64), pairs grouped by polygon id (untimed), "
                         f"one *_contains_batch call per polygon, polygons split over {th} "
                         f"threads, 3 engines; second of two full passes, {t * 1e3:.1f} ms",
               "per_pair_scalar": {"value": 3 * m / (sum(sc) * 1e-9), "unit": UNIT, "cores": th,
                                   "what": "the reference's early-exit scalar tests on every "
                                           "pair in stream order (random polygon ids), "
                                           f"{th} threads"}}
        par["vs_reference"] = block(words, rw, xs, ys, BC.EPS32, join=(job.off, ids))
    elif job.f64 and job.workload == "c1":
        ns, masks, build, (vx, vy, xs, ys) = reference_c1(th)
        ns, masks, build, _ = reference_c1(th)
        t = sum(ns) * 1e-9
        rw = [np.pad(np.packbits(mk, bitorder="little"), (0, (-((m + 7) // 8)) % 4)).view(np.uint32)
              for mk in masks]
        cpu = {"value": 3 * m / t, "unit": UNIT, "cores": th, "kind": "reference",
               "sample": f"the unmodified reference library ({build}), all {m} f64 points, 3 "
                         f"engines *_contains_batch(threads={th}); second of two passes"}
        par["vs_reference"] = block(words, rw, xs, ys, BC.EPS64)
    else:
        # (f64 runs: the widened f32 stream, so .float() is exact)
        xs, ys = job.xs.float().cpu().numpy(), job.ys.float().cpu().numpy()
        rr = BC.RefRun(job.vx, job.vy, xs, ys, th)
        res = rr.run(packed=True)  # warm-up pass: the reference masks
        timed = [rr.run() for _ in range(CPU_PASSES)]  # the timed passes
        rr.close()
        ts = [sum(x["ns"] for x in r) * 1e-9 for r in timed]
        t = statistics.median(ts)
        res2 = timed[ts.index(t)] if t in ts else timed[-1]
        cpu = {"value": 3 * m / t, "unit": UNIT, "cores": th, "kind": "reference",
               "sample": rr.describe() + f"; median of {CPU_PASSES} full passes after one "
                                         f"warm-up pass, {t * 1e3:.1f} ms",
               "pass_ms": [round(x * 1e3, 1) for x in ts],
               "count_inside_ms": sum(x["count_ns"] for x in res2) * 1e-6,
               "inside_counts": [x["inside"] for x in res2]}
        rw = [x["words"] for x in res]
        par["vs_reference"] = block(words, rw, xs, ys, BC.EPS64 if job.f64 else BC.EPS32)
        if job.f64:  # the step itself ran the exact kernels: bit-exact or nothing
            par["outside_band"] = sum(v["outside_band"] for v in par["vs_reference"].values())
            return cpu, par
        # the reference-exact f64 kernels over the whole batch, on the device
        xd, yd = job.xs.double(), job.ys.double()
        w64 = [torch.zeros_like(w) for w in words]
        job.poly.test_multi(xd, yd, (0, 1, 2), words=w64)
        torch.cuda.synchronize()
        del xd, yd
        par["f32_vs_f64_exact"] = block(words, w64, xs, ys, BC.EPS32)
        par["f64_exact_vs_reference"] = block(w64, rw, xs, ys, BC.EPS64)
        del w64
    par["outside_band"] = sum(v["outside_band"] for k, blk in par.items() if isinstance(blk, dict)
                              for v in blk.values())
    return cpu, par


# ----------------------------------------------------------------- GPU arm
def stdout_to_stderr(fn, *a):
    """Run fn with fd 1 pointed at stderr: NCCL prints its version banner on
    stdout at communicator init, and stdout must carry exactly one JSON line."""
    sys.stdout.flush()
    saved = os.dup(1)
    os.dup2(2, 1)
    try:
        return fn(*a)
    finally:
        os.dup2(saved, 1)
        os.close(saved)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-convert", action="store_true")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"],
                    help="f64: the workload's points widened exactly to f64 and tested by the "
                         "reference-exact f64 kernels (the reference's own precision)")
    ap.add_argument("--fused", action="store_true",
                    help="(default for f32 single-polygon workloads) one fused kernel for the "
                         "three engines (vpipg_test_multi)")
    ap.add_argument("--separate", action="store_true",
                    help="three per-engine kernels per step instead of the fused one")
    ap.add_argument("--no-graph", action="store_true",
                    help="time eager launches instead of CUDA-graph replays of the step")
    ap.add_argument("--points", type=int, default=0, help="override the workload size (profiling)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank, world = env_int("RANK", 0), env_int("WORLD_SIZE", 1)
    local = env_int("LOCAL_RANK", 0)
    if args.gpus > 1 and "RANK" not in os.environ:
        # `python bench.py --gpus N` on its own: relaunch as N ranks (one per GPU)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                  "--master-port", str(port), str(Path(__file__).resolve()),
                                  *sys.argv[1:]])
    if world != args.gpus and rank == 0:
        print(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}",
              file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2007_15385_b200 as vp
    from paper_2007_15385_b200.multi import CountComm

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    # the count all-reduce: libvpipg's own NCCL communicator on the launch
    # stream (a 1-rank communicator at N=1, so the step is the same at every N)
    comm = stdout_to_stderr(CountComm.from_process_group, local)
    M = args.points or workload_size(args.workload)
    lo, hi = W.shard(M, rank, world)
    m = hi - lo
    with torch.cuda.stream(stream):
        job = (JoinJob if args.workload == "c4" else PolygonJob)(args.workload, lo, hi, local,
                                                                 torch, vp, stream, args.dtype)
        words = [torch.zeros((m + 31) // 32, dtype=torch.int32, device="cuda") for _ in range(3)]
        counts = torch.zeros(3, dtype=torch.int64, device="cuda")
        flush = torch.ones(256 << 20, dtype=torch.uint8, device="cuda") if M * 8 <= 4 * 126e6 else None
        flush_sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    stream.synchronize()
    n_edges = job.n_edges
    # the three engines in one kernel that reads every point once (f32, one
    # polygon); the per-engine kernels are still timed below for the breakdown
    if isinstance(job, JoinJob):  # the join fuses whenever all three engines run
        fused = not args.separate
    else:
        fused = (not args.separate) and job.poly.multi_fused(job.xs, job.ys)  # the library's plan

    kevents = []  # per step, per engine: (start, end) on the launch stream
    sevents = []  # per step: (start, end) around the step's own work, flush excluded

    def step(record: bool):
        if flush is not None:
            # L2 flush by READING a 256 MB buffer (clean lines: no write-back
            # traffic leaks into the timed kernels); outside the step's events
            flush_sink.copy_(flush.view(torch.int64).sum(dtype=torch.int64).view(1))
        if record:
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
        vp.zero_counts(counts, stream)
        pairs = []
        if fused:  # one kernel: its time is reported once, for all three engines
            if record:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            job.launch_all(words, [counts[e:e + 1] for e in range(3)], stream)
            if record:
                b.record(stream)
                pairs = [(a, b)] * 3
        for e in range(0 if fused else 3):
            if record:
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
            job.launch(e, words[e], counts[e:e + 1], stream)
            if record:
                b.record(stream)
                pairs.append((a, b))
        comm.allreduce(counts, stream)  # NCCL sum of the 3 inside counts
        if record:
            s1.record(stream)
            kevents.append(pairs)
            sevents.append((s0, s1))

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step(False)
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        # the step's work (count reset, 3 engine launches, count all-reduce) as
        # one CUDA graph; the per-kernel times come from K eager steps run just
        # before the timed graph replays (events cannot sit inside the graph)
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                step(True)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            vp.zero_counts(counts, stream)
            if fused:
                job.launch_all(words, [counts[e:e + 1] for e in range(3)], stream)
            else:
                for e in range(3):
                    job.launch(e, words[e], counts[e:e + 1], stream)
            comm.allreduce(counts, stream)
        with torch.cuda.stream(stream):
            for _ in range(2):
                graph.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gpus = os.environ.get("CUDA_VISIBLE_DEVICES", ",".join(str(i) for i in range(world)))
    sampler = ClockSampler(gpus if rank == 0 else str(local)) if rank == 0 else None
    time.sleep(0.2 if rank == 0 else 0)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    gevents = []  # graph mode: per step (start, end) around the replay, flush excluded
    with torch.cuda.stream(stream):
        t_start.record(stream)
        for _ in range(args.steps):
            if graph is None:
                step(True)
                continue
            if flush is not None:
                flush_sink.copy_(flush.view(torch.int64).sum(dtype=torch.int64).view(1))
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record(stream)
            graph.replay()
            g1.record(stream)
            gevents.append((g0, g1))
        t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    if graph is not None:
        sevents = gevents
    # K steps bracketed by t_start / t_end; with an L2 flush between steps the
    # flush kernels sit inside that bracket, so the sum of the per-step events
    # (each starting after its flush) is the timed work instead
    ms = (t_start.elapsed_time(t_end) if flush is None
          else sum(a.elapsed_time(b) for a, b in sevents))
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    per_kernel_ms = [statistics.mean(p[e][0].elapsed_time(p[e][1]) for p in kevents)
                     for e in range(3)]
    final_counts = counts.tolist()
    sep_ms = None
    if fused:
        # per-engine breakdown: K eager steps of the three separate kernels
        # (same inputs, same flush), outside the timed region, after one
        # untimed pass (their first launches load the kernels' modules)
        sep = []
        with torch.cuda.stream(stream):
            vp.zero_counts(counts, stream)
            for e in range(3):
                job.launch(e, words[e], counts[e:e + 1], stream)
            for _ in range(args.steps):
                if flush is not None:
                    flush_sink.copy_(flush.view(torch.int64).sum(dtype=torch.int64).view(1))
                vp.zero_counts(counts, stream)
                ev = []
                for e in range(3):
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    job.launch(e, words[e], counts[e:e + 1], stream)
                    b.record(stream)
                    ev.append((a, b))
                sep.append(ev)
        torch.cuda.synchronize()
        sep_ms = [statistics.mean(p[e][0].elapsed_time(p[e][1]) for p in sep) for e in range(3)]
        assert counts.tolist() == final_counts or world > 1  # same answers as the fused kernel

    # ---- end-to-end through the public API with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        job.prepare_host()
        hw = [torch.empty((m + 31) // 32, dtype=torch.int32, pin_memory=True) for _ in range(3)]
        torch.cuda.synchronize()
        times = []
        for r in range(1 + args.e2e_steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            cnt = job.run_host(hw, stream)
            if world > 1:
                ct = torch.tensor(cnt, dtype=torch.int64, device="cuda")
                dist.all_reduce(ct)
                ct.cpu()
            dt = time.perf_counter() - t0
            if r > 0:
                times.append(dt)
        t_e2e = torch.tensor([statistics.mean(times)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
        e2e = {"value": 3 * M / float(t_e2e.item()), "unit": UNIT,
               "h2d_bytes_per_step": job.bytes_per_unit * m,
               "d2h_bytes_per_step": 3 * 4 * ((m + 31) // 32),
               "steps": args.e2e_steps, "step_ms": [round(t * 1e3, 2) for t in times],
               "path": job.e2e_path}

    cpu = parity = convert = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the e2e leg's pinned host copies of the inputs (17 GB at C5) go back to
        # the OS first: the reference's threads should find the host as the
        # reference arm's own process does
        job.release_host()
        hw = None
        getattr(torch._C, "_host_emptyCache", lambda: None)()
        cpu, parity = cpu_leg(job, words, m, torch)
    if rank == 0 and not args.no_convert:
        convert = convert_block(vp, local, stream)

    if world > 1:
        dist.barrier()
    del graph  # its NCCL node references the communicator: release it first
    comm.close()  # every rank is past its last count all-reduce
    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return

    hbm_peak, hbm_src, fma_peak = load_peaks()
    bytes_per_launch = m * job.bytes_per_unit + 4 * ((m + 31) // 32)
    pe = int(m * n_edges)
    clk_hz = ((clocks or {}).get("sm_mhz") or 1965.0) * 1e6
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    f64 = getattr(job, "f64", False)
    names = ("voronoi", "sign_of_offset", "ray_crossing")
    words_bytes = 4 * ((m + 31) // 32)

    def kernel_entry(name, ms_k, engines):
        """One kernel's rates: `engines` = the engine names it runs (3 for the fused one)."""
        t = ms_k * 1e-3
        nbytes = bytes_per_launch + (len(engines) - 1) * words_bytes
        k = {"engine": name, "ms": ms_k, "GB_per_s": nbytes / t / 1e9,
             "point_edge_per_s": len(engines) * pe / t,
             "tflops_alg": 4 * len(engines) * pe / t / 1e12}
        if job.issue_cycles:
            cyc = sum(job.issue_cycles[e] for e in engines) / len(engines)
            k["issue_model_frac"] = k["point_edge_per_s"] / (sms * 4 * 32 * clk_hz / cyc)
        return k

    if fused:
        kernels = [kernel_entry("fused", per_kernel_ms[0], names)]
        per_kernel_ms = per_kernel_ms[:1]
        engines_separate = [kernel_entry(n, sep_ms[e], (n,)) for e, n in enumerate(names)]
    else:
        kernels = [kernel_entry(n, per_kernel_ms[e], (n,)) for e, n in enumerate(names)]
        engines_separate = None
    n_eng = 3 if fused else 1  # engine tests per point in one launch of the dominant kernel
    alg_bytes = bytes_per_launch + (n_eng - 1) * words_bytes
    dom = max(range(len(kernels)), key=lambda e: per_kernel_ms[e])
    dk = kernels[dom]
    hbm_frac = dk["GB_per_s"] / hbm_peak
    fma_tflops = 2 * fma_peak / 1e12 if fma_peak else 2 * FFMA_PER_SM_CLK * 148 * 1.965e9 / 1e12
    if f64:  # DFMA issues at half the FFMA rate (profiles/pipe_peaks_r01.json)
        fma_tflops /= 2
    fma_frac = dk["tflops_alg"] / fma_tflops
    compute_bound = (4 * n_eng * pe / (fma_tflops * 1e12)) > (alg_bytes / (hbm_peak * 1e9))
    traffic = None
    try:  # DRAM bytes per launch from the committed ncu --set full capture (same kernel/config)
        tj = json.loads(TRAFFIC_FILE.read_text())[args.workload + ("f64" if f64 else "")]
        traffic = tj["dram_bytes_per_launch"][dk["engine"]] * m / tj["points"]
    except Exception:
        pass
    if f64:
        # the exact kernels issue the reference's DADD / DMUL / DSETP sequence:
        # their bound is the FP64 pipe (2 dispatch cycles per instruction)
        cyc = sum(job.issue_cycles[e] for e in names if (dk["engine"] == "fused" or e == dk["engine"]))
        achieved = (cyc / 2) * pe / 32 / (per_kernel_ms[dom] * 1e-3) / 1e12
        peak = sms * 4 * clk_hz / 2 / 1e12
        roof = {"bound": "fp64-pipe", "achieved": achieved, "peak": peak,
                "unit": "T FP64 warp-instructions/s", "frac": achieved / peak, "traffic": traffic}
    elif compute_bound:
        roof = {"bound": "fp64-fma" if f64 else "fp32-fma", "achieved": dk["tflops_alg"],
                "peak": fma_tflops,
                "unit": "TFLOP/s", "frac": fma_frac, "traffic": traffic}
    else:
        roof = {"bound": "hbm", "achieved": dk["GB_per_s"], "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm_frac, "traffic": traffic}
    roof.update({"kernel": dk["engine"], "hbm_GB_per_s": dk["GB_per_s"], "hbm_frac": hbm_frac,
                 "hbm_peak_source": hbm_src, "fma_frac": fma_frac,
                 "fma_peak_source": "tools/pipe_peaks.cu FFMA lane-ops/s x2 (profiles/pipe_peaks_r01.json)",
                 "per_unit": (f"{alg_bytes / m:.3f} B and {4 * n_edges * n_eng} flops per point "
                              f"({n_eng} engine test(s), n={n_edges} edges, 4 flops per "
                              f"point-edge)"),
                 "algorithmic_bytes_per_launch": alg_bytes,
                 "traffic_source": "profiles/traffic_r02.json (ncu --set full dram__bytes_read+write "
                                   "of this kernel on this workload, scaled to this launch)",
                 "issue_model_frac": dk.get("issue_model_frac"),
                 "issue_model": ("FP64-pipe cycles per point-edge (2 per DADD / DMUL / DSETP): "
                                 "Voronoi 12, offset 8, crossing 14 "
                                 "(profiles/ncu_full_r02_c5f64.json)" if f64 else
                                 "dispatch cycles per point-edge: slab 2 (FFMA + FMNMX3/2), "
                                 "crossing 5.5 (1.5 FADD + FFMA + 1.5 LOP3, paired anchoring); the "
                                 "fused kernel their mean over the three engines; "
                                 "profiles/crossing_forms_r02.json")})
    try:  # the ncu evidence for the same kernel and workload (issue / pipe utilisation)
        nk = json.loads(NCU_FILE.with_name(
            f"ncu_full_r02_{args.workload.replace(':', 'n')}{'f64' if f64 else ''}.json")
                        .read_text())["kernels"][dk["engine"] + ("_f64" if f64 else "")]
        roof["ncu"] = {k.split(".")[0]: nk[k] for k in (
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active") if k in nk}
    except Exception:
        pass

    step_s = ms_max * 1e-3 / args.steps
    total_tests = 3 * M
    line = {
        "metric": METRIC, "value": total_tests / step_s, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if f64 else "f32",
        "data": "synthetic (seeded counter-based points, reference-sampler polygon)",
        "config": config_block(args, world),
        "execution": {"n_edges": n_edges,
                   "engines_fused": fused,
                   "launch": ("eager launches" if args.no_graph else
                              "one CUDA-graph replay per step (" +
                              ("the fused three-engine kernel" if fused else "3 engine kernels") +
                              " + count all-reduce); per-kernel times from K eager steps before "
                              "it" + ("; engines_separate: K eager steps of the three "
                                      "per-engine kernels after it" if fused else ""))},
        "gpu_launches": (1 if fused else 3) * args.steps,
        "roofline": roof, "kernels": kernels, "engines_separate": engines_separate,
        "inside_counts": final_counts,
        "prepare_ms": job.prep_ms,
        "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu, "parity": parity, "convert": convert,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
