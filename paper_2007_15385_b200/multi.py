"""Multi-GPU host logic: point shards + the one count all-reduce.

The batch is partitioned into contiguous, `align`-point-aligned ranges (one
per rank). With `align` a multiple of 32, each rank's PIPM mask words start at
word `lo // 32` of the global mask, so per-rank masks concatenate without bit
shifts (the multi-GPU analogue of the reference's thread chunking,
engines.cpp:30-52; masks never depend on the partitioning,
test_engines.cpp:227-241). The only exchanged data is the vector of inside
counts (one u64 per engine), summed with one all-reduce: on GPUs the
library's own NCCL communicator (`CountComm`, vpipg_allreduce_counts, launched
on the kernels' stream), in the CPU tests torch.distributed over gloo.
"""
from __future__ import annotations

import ctypes as C

from ._lib import check, load


def shard(m: int, rank: int, world: int, align: int = 1024) -> tuple[int, int]:
    """[lo, hi) of rank `rank`: contiguous, lo a multiple of `align`."""
    if world < 1 or not 0 <= rank < world or align % 32:
        raise ValueError("bad shard request")
    per = -(-m // world)
    per = -(-per // align) * align
    lo = min(m, rank * per)
    return lo, min(m, lo + per)


def reduce_counts(counts, group=None):
    """Sum the per-rank inside counts in place (int64 tensor) across the group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def shared_unique_id(group=None) -> bytes:
    """An NCCL unique id made on rank 0 and broadcast to every rank of `group`."""
    import torch.distributed as dist
    obj = [CountComm.unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class CountComm:
    """The library's NCCL communicator for the count all-reduce (vpipg_comm_*).

    torch.distributed is only the out-of-band channel for the 128-byte NCCL
    unique id (`from_process_group`); the collective itself is issued by
    libvpipg on the caller's stream."""

    def __init__(self, uid: bytes, nranks: int, rank: int, device: int):
        self._h = C.c_void_p()
        check(load().vpipg_comm_init(uid, nranks, rank, device, C.byref(self._h)),
              "vpipg_comm_init")
        self.nranks, self.rank, self.device = nranks, rank, device

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(load().vpipg_comm_unique_id(buf), "vpipg_comm_unique_id")
        return buf.raw

    @staticmethod
    def nccl_version() -> int:
        v = C.c_int()
        check(load().vpipg_nccl_version(C.byref(v)), "vpipg_nccl_version")
        return v.value

    @classmethod
    def from_process_group(cls, device: int, group=None) -> "CountComm":
        """Rank 0 makes the id; the process group broadcasts it; every rank joins."""
        import torch.distributed as dist
        if not (dist.is_available() and dist.is_initialized()):
            return cls(cls.unique_id(), 1, 0, device)
        uid = shared_unique_id(group)
        return cls(uid, dist.get_world_size(group), dist.get_rank(group), device)

    def allreduce(self, counts, stream=None) -> None:
        """In-place sum of a device int64/uint64 tensor of counts, on `stream`."""
        s = stream.cuda_stream if stream is not None else None
        check(load().vpipg_allreduce_counts(self._h, C.c_void_p(counts.data_ptr()),
                                            counts.numel(), C.c_void_p(s)),
              "vpipg_allreduce_counts")

    def close(self) -> None:
        if self._h:
            check(load().vpipg_comm_destroy(self._h), "vpipg_comm_destroy")
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
