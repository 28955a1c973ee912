"""Multi-GPU plumbing: one process per GPU, NCCL communicator inside the C
ABI (gd_comm_*), torch.distributed only to broadcast the 128-byte NCCL id.

Sharding: every rank holds a replica of the store and applies
every batch; PageRank pulls only its destination range and all-gathers the
rank vector each sweep; TC counts a contiguous 1/world slice of each phase's
records and all-reduces the count delta.  `ShardPlan` is the partition the
device code uses (csrc/gd_comm.cuh: chunk = ceil(n / world)); the CPU tests
drive it with gloo.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _native as N


@dataclass(frozen=True)
class ShardPlan:
    """1D block ownership of the vertex ids, as the device code uses it
    (csrc/gd_comm.cuh Blocks): the reference's block_ranges
    (partition.py:69-78) -- the first n % world ranks get one vertex more."""

    n: int
    world: int

    @property
    def chunk(self) -> int:
        """The largest block (the padded per-rank size of a reduce-scatter)."""
        return self.n // self.world + (1 if self.n % self.world else 0)

    @property
    def padded(self) -> int:
        return self.chunk * self.world

    def range(self, rank: int):
        base, rem = divmod(self.n, self.world)
        lo = rank * base + min(rank, rem)
        return lo, lo + base + (1 if rank < rem else 0)

    def owner(self, v):
        """Owner rank of vertex id(s) v (scalar or numpy array)."""
        import numpy as np

        base, rem = divmod(self.n, self.world)
        big = rem * (base + 1)
        v = np.asarray(v)
        return np.where(v < big, v // (base + 1), rem + (v - big) // max(base, 1))

    def record_slice(self, k: int, rank: int):
        """Contiguous slice of k batch records counted by `rank` (TC)."""
        return k * rank // self.world, k * (rank + 1) // self.world


def unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    N.check(N.lib().gd_comm_unique_id(buf))
    return bytes(buf)


class Communicator:
    """NCCL communicator owned by the C ABI."""

    def __init__(self, world: int, rank: int, nccl_id: bytes, device: int = 0, *, _handle=None):
        if _handle is None:
            buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            h = C.c_void_p()
            N.check(N.lib().gd_comm_create(int(world), int(rank), buf, int(device), C.byref(h)))
        else:
            h = _handle
        self.h = h
        self.world = world
        self.rank = rank

    @classmethod
    def local_group(cls, world: int, device: int = 0, group: int = 0) -> list:
        """`world` members of an in-process group (gd_comm_create_local): one
        per host thread, all on `device` -- the partitioned code paths on a
        single GPU, for tests."""
        out = []
        for r in range(world):
            h = C.c_void_p()
            N.check(N.lib().gd_comm_create_local(int(world), r, int(group), int(device), C.byref(h)))
            out.append(cls(world, r, b"", device, _handle=h))
        return out

    @classmethod
    def from_torch_distributed(cls, device: int) -> "Communicator":
        import torch.distributed as dist

        obj = [unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls(dist.get_world_size(), dist.get_rank(), obj[0], device)

    def attach(self, algo) -> None:
        """Shard a PRHandle / TCHandle over this communicator."""
        fn = {"pr": "gd_pr_set_comm", "tc": "gd_tc_set_comm"}.get(algo.kind)
        if fn is None:
            raise ValueError(f"{algo.kind} handles run as replicas (no sharded path)")
        N.check(getattr(N.lib(), fn)(algo.h, self.h))
        algo.comm = self  # keep alive

    def stats(self) -> dict:
        """Communication accounting since creation / reset (CommStats analogue)."""
        import numpy as np

        out = np.zeros(5, dtype=np.int64)
        N.check(N.lib().gd_comm_stats_ex(self.h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return {"calls": int(out[0]), "allgather_bytes": int(out[1]), "allreduce_bytes": int(out[2]),
                "sent_bytes": int(out[3]), "alltoall_bytes": int(out[4])}

    def reset_stats(self) -> None:
        N.check(N.lib().gd_comm_reset_stats(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and N._lib is not None:
            N._lib.gd_comm_destroy(h)
            self.h = None
