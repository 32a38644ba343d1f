"""World-size-2 gloo test of the multi-GPU host logic (CPU only).

Each rank takes its shard of a C5-style counter point stream, computes its
masks (the CPU oracle stands in for the per-GPU kernels here: this test checks
the sharding and the collective, the GPU tests check the kernels), and the
inside counts are all-reduced with the same helper bench.py uses. Rank 0 checks
that the concatenated per-rank mask words equal the single-process masks and
that the reduced counts equal the global counts.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W
from paper_2007_15385_b200.multi import reduce_counts, shard, shared_unique_id


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, m, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    orc = oracle.Oracle()
    vx, vy = W.c5_polygon(orc.random_convex_polygon)
    lo, hi = shard(m, rank, world)
    xs, ys = orc.counter_points_f32(W.c5_point_seed(), lo, hi - lo, W.C5_BOX)
    masks = orc.masks(vx, vy, xs.astype(np.float64), ys.astype(np.float64))
    words = [np.packbits(mk, bitorder="little") for mk in masks]
    counts = torch.tensor([int(mk.sum()) for mk in masks], dtype=torch.int64)
    reduce_counts(counts)
    # the NCCL unique id of the library's count communicator travels over the
    # process group; every rank must hold rank 0's bytes
    uid = shared_unique_id()
    gathered = [None] * world
    dist.all_gather_object(gathered, (lo, hi, words, uid))
    if rank == 0:
        out.put((counts.tolist(), gathered))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [1 << 16, (1 << 16) + 12345])
def test_two_rank_shards_and_count_allreduce(m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, m, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, gathered = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import oracle
    orc = oracle.Oracle()
    vx, vy = W.c5_polygon(orc.random_convex_polygon)
    xs, ys = orc.counter_points_f32(W.c5_point_seed(), 0, m, W.C5_BOX)
    full = orc.masks(vx, vy, xs.astype(np.float64), ys.astype(np.float64))
    assert counts == [int(mk.sum()) for mk in full]
    (lo0, hi0, w0, u0), (lo1, hi1, w1, u1) = gathered
    assert len(u0) == 128 and u0 == u1
    assert lo0 == 0 and hi0 == lo1 and hi1 == m and lo1 % 1024 == 0
    for e in range(3):
        # shard boundaries are 32-aligned, so the packed masks simply concatenate
        cat = np.concatenate([w0[e], w1[e]])
        assert np.array_equal(cat, np.packbits(full[e], bitorder="little"))


def test_shard_properties():
    for m in (0, 1, 31, 1024, 10**6 + 7, 1 << 31):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard(m, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == m
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            for a, b in ranges:
                assert (a % 1024 == 0 or a == b == m) and a <= b
    with pytest.raises(ValueError):
        shard(10, 0, 2, align=48)


def test_bench_reference_arm_two_ranks_under_torchrun():
    """The driver's N > 1 launch path, end to end on the CPU: `bench.py --gpus 2`
    relaunches itself under torch.distributed.run (127.0.0.1), rank 0 runs the
    reference arm on the full (here: reduced) config and prints ONE JSON line,
    rank 1 exits 0 without work."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    import oracle
    try:
        oracle.Reference()
    except FileNotFoundError:
        pytest.skip("oracle/_ref not built")
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--points", str(1 << 16), "--steps", "1", "--warmup", "1"],
                         cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["config"]["points"] == 1 << 16
