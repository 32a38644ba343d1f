"""World-size-2 run of the sharded step with the real kernels (B200).

The N > 1 path of bench.py splits the C5 point stream into contiguous,
1024-aligned shards (`multi.shard`); every rank generates its own shard on its
GPU (`fill_uniform_points` from the shard's first index), runs the fused
three-engine kernel on it and all-reduces the three inside counts. Only one
GPU is available here, so both ranks run their (independent) kernels on
cuda:0 and the count all-reduce and the mask gather travel over gloo on the
host -- no kernel waits on another rank's work. Rank 0 checks that the
concatenated per-rank words and the reduced counts equal one single-process
pass over the whole batch.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_shard(vp, lo, hi):
    """Words (three u32 arrays) and counts of the fused pass over [lo, hi)."""
    m = hi - lo
    xs = torch.empty(m, dtype=torch.float32, device=DEV)
    ys = torch.empty_like(xs)
    vp.fill_uniform_points(W.c5_point_seed(), lo, xs, ys, W.C5_BOX)
    vx, vy = W.c5_polygon(vp.random_convex_polygon)
    ws = [torch.zeros((m + 31) // 32, dtype=torch.int32, device=DEV) for _ in range(3)]
    cs = torch.zeros(3, dtype=torch.int64, device=DEV)
    with vp.PreparedPolygon.prepare(vx, vy, vp.KIND_ALL) as p:
        assert p.multi_fused(xs, ys) or m < (1 << 14)
        p.test_multi(xs, ys, words=ws, counts=[cs[e:e + 1] for e in range(3)])
        torch.cuda.synchronize()
    return [w.cpu().numpy().view(np.uint32) for w in ws], cs.cpu()


def _rank(rank, world, port, m, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2007_15385_b200 as vp
    from paper_2007_15385_b200.multi import reduce_counts, shard
    torch.cuda.set_device(0)
    lo, hi = shard(m, rank, world)
    words, counts = _run_shard(vp, lo, hi)
    reduce_counts(counts)
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, words))
    if rank == 0:
        out.put((counts.tolist(), gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [1 << 22, (1 << 22) + 777])
def test_two_rank_sharded_fused_pass_equals_one_pass(m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, m, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import paper_2007_15385_b200 as vp
    full_words, full_counts = _run_shard(vp, 0, m)
    assert counts == full_counts.tolist()
    (lo0, hi0, w0), (lo1, hi1, w1) = gathered
    assert lo0 == 0 and hi0 == lo1 and hi1 == m and lo1 % 1024 == 0
    for e in range(3):
        # 1024-aligned shard starts: the per-rank words simply concatenate
        assert np.array_equal(np.concatenate([w0[e], w1[e]]), full_words[e]), e
