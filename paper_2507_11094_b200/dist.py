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
    n: int
    world: int

    @property
    def chunk(self) -> int:
        return (self.n + self.world - 1) // self.world if self.world else self.n

    @property
    def padded(self) -> int:
        return self.chunk * self.world

    def range(self, rank: int):
        lo = min(self.n, rank * self.chunk)
        return lo, min(self.n, lo + self.chunk)

    def record_slice(self, k: int, rank: int):
        """Contiguous slice of k batch records counted by `rank` (TC)."""
        return k * rank // self.world, k * (rank + 1) // self.world


def unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    N.check(N.lib().gd_comm_unique_id(buf))
    return bytes(buf)


class Communicator:
    """NCCL communicator owned by the C ABI."""

    def __init__(self, world: int, rank: int, nccl_id: bytes, device: int = 0):
        buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        N.check(N.lib().gd_comm_create(int(world), int(rank), buf, int(device), C.byref(h)))
        self.h = h
        self.world = world
        self.rank = rank

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

        out = np.zeros(4, dtype=np.int64)
        N.check(N.lib().gd_comm_stats(self.h, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return {"calls": int(out[0]), "allgather_bytes": int(out[1]), "allreduce_bytes": int(out[2]),
                "sent_bytes": int(out[3])}

    def reset_stats(self) -> None:
        N.check(N.lib().gd_comm_reset_stats(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and N._lib is not None:
            N._lib.gd_comm_destroy(h)
            self.h = None
