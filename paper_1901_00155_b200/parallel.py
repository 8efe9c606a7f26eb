"""Several GPUs: candidates sharded, best-so-far max-reduced.

Every rank holds the whole prepared series (preparation is replicated: it takes
milliseconds and avoids moving the matrix).  Entry ``e`` of the rarity order belongs
to rank ``e mod world``.  After every outer-loop batch the ranks max-reduce two packed
64-bit keys: the best-so-far ``(float bits of d^2) << 32 | ~row`` — integer max is
"greater distance, then smaller position", the reference's deterministic merge rule
(discovery.cpp:328-340) — and a "some rank still has candidates" flag that ends the loop
on all ranks together (one 16-byte ``ncclAllReduce(ncclMax, ncclUint64)`` per batch) —
and, unless the engine option ``share_bounds`` is off, min-reduce the N packed nn bounds
(``ncclAllReduce(ncclMin, ncclUint64, N)``), so that what one rank's scans learn about a
row prunes it on every rank.

Two transports:
  * ``attach_nccl``   the engine's own NCCL communicator (libnccl loaded by the C library);
                      torch.distributed only carries the 128-byte unique id.
  * ``attach_torch``  a host hook that calls ``torch.distributed.all_reduce(MAX)`` —
                      works on gloo (CPU tests) and nccl alike.
"""
from __future__ import annotations

import numpy as np

INF_BITS = 0x7F800000


def owner_of(entry: int, world: int) -> int:
    """Rank that scans entry ``entry`` of the rarity order."""
    return entry % world


def pack_best(d2: float, row: int) -> int:
    """Packed best-so-far key of a squared distance (float32, >= 0) and a 0-based row."""
    bits = int(np.float32(d2).view(np.uint32))
    return (bits << 32) | (0xFFFFFFFF - row)


def unpack_best(key: int) -> tuple[float, int]:
    bits = np.uint32(key >> 32)
    return float(bits.view(np.float32)), 0xFFFFFFFF - (key & 0xFFFFFFFF)


class TorchExchange:
    """In-place element-wise max of uint64 keys over a torch.distributed group.

    Keys never have bit 63 set (float bits of a non-negative number are < 2^31), so they
    are exchanged as int64 without changing their order."""

    def __init__(self, group=None, device="cpu"):
        import torch
        import torch.distributed as dist

        self._torch, self._dist, self._group, self._device = torch, dist, group, device
        self.calls = 0

    def __call__(self, keys: np.ndarray) -> None:
        torch, dist = self._torch, self._dist
        if int(keys.max(initial=0)) >> 63:
            raise ValueError("packed keys must stay below 2^63")
        t = torch.from_numpy(keys.view(np.int64).copy()).to(self._device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self._group)
        keys[:] = t.cpu().numpy().view(np.uint64)
        self.calls += 1


def attach_torch(ctx, group=None, device="cpu") -> TorchExchange:
    import torch.distributed as dist

    ex = TorchExchange(group, device)
    ctx.set_exchange(ex, dist.get_world_size(group), dist.get_rank(group))
    return ex


def attach_nccl(ctx, group=None) -> None:
    """Creates the engine's NCCL communicator; rank 0's unique id travels over ``group``."""
    import torch.distributed as dist

    from .engine import comm_unique_id

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    box = [comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    ctx.comm_init(box[0], world, rank)
