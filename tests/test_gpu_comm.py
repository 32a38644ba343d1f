"""The library's own count all-reduce on a B200 (vpipg_comm_*).

Only one GPU is available to the tests, so the communicators here have one
rank; the multi-rank id exchange and shard logic are covered on the CPU by
tests/test_multi_rank.py (gloo, world size 2)."""
import ctypes as C

import numpy as np
import pytest
import torch

import workloads as W
import paper_2007_15385_b200 as vp
from paper_2007_15385_b200 import _lib
from paper_2007_15385_b200.multi import CountComm

pytestmark = pytest.mark.gpu


def test_one_rank_comm_on_the_kernel_stream():
    s = torch.cuda.Stream()
    vx, vy = W.c1_polygon()
    m = 1 << 22
    xs = torch.empty(m, dtype=torch.float32, device="cuda")
    ys = torch.empty_like(xs)
    vp.fill_uniform_points(11, 0, xs, ys, W.C1_BOX)
    torch.cuda.synchronize()
    assert CountComm.nccl_version() >= 21800
    with CountComm(CountComm.unique_id(), 1, 0, 0) as comm, \
            vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        counts = torch.zeros(3, dtype=torch.int64, device="cuda")
        ref = []
        for e in range(3):
            c = torch.zeros(1, dtype=torch.int64, device="cuda")
            p.test(e, xs, ys, count=c)
            torch.cuda.synchronize()
            ref.append(int(c.item()))
        with torch.cuda.stream(s):
            for e in range(3):
                p.test(e, xs, ys, count=counts[e:e + 1], stream=s)
            comm.allreduce(counts, s)
        s.synchronize()
        assert counts.tolist() == ref and min(ref) > 0


def test_init_all_and_grouped_allreduce():
    lib = _lib.load()
    devs = (C.c_int * 1)(0)
    comms = (C.c_void_p * 1)()
    assert lib.vpipg_comm_init_all(1, devs, comms) == 0
    nr, rk, dv = C.c_int(), C.c_int(), C.c_int()
    assert lib.vpipg_comm_info(comms[0], C.byref(nr), C.byref(rk), C.byref(dv)) == 0
    assert (nr.value, rk.value, dv.value) == (1, 0, 0)
    t = torch.tensor([5, 7, 1 << 40], dtype=torch.int64, device="cuda")
    ptrs = (C.c_void_p * 1)(t.data_ptr())
    streams = (C.c_void_p * 1)(torch.cuda.current_stream().cuda_stream)
    assert lib.vpipg_allreduce_counts_group(1, comms, ptrs, 3, streams) == 0
    torch.cuda.synchronize()
    assert t.tolist() == [5, 7, 1 << 40]
    assert lib.vpipg_comm_destroy(comms[0]) == 0


def test_step_is_graph_capturable():
    """The bench step -- three engine launches plus the count all-reduce on one
    stream -- captures into a CUDA graph and replays with identical results."""
    vx, vy = W.c5_polygon(vp.random_convex_polygon)
    m = (1 << 22) + 777
    xs = torch.empty(m, dtype=torch.float32, device="cuda")
    ys = torch.empty_like(xs)
    vp.fill_uniform_points(W.c5_point_seed(), 0, xs, ys, W.C5_BOX)
    words = [torch.zeros((m + 31) // 32, dtype=torch.int32, device="cuda") for _ in range(3)]
    counts = torch.zeros(3, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    with CountComm(CountComm.unique_id(), 1, 0, 0) as comm, \
            vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        def step():
            counts.zero_()
            for e in range(3):
                p.test(e, xs, ys, words=words[e], count=counts[e:e + 1], stream=s)
            comm.allreduce(counts, s)

        with torch.cuda.stream(s):
            step()  # eager reference (also warms the launch path up)
        s.synchronize()
        ref_words = [w.clone() for w in words]
        ref_counts = counts.clone()
        for w in words:
            w.zero_()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        assert counts.tolist() == ref_counts.tolist()
        for w, r in zip(words, ref_words):
            assert torch.equal(w, r)
