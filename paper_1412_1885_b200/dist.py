"""Multi-GPU plumbing: slab partition of Y along its last mode and the cross-rank reduction
hook of the C-ABI (tk_comm), over torch.distributed (NCCL on B200s, gloo on CPU tests).

Semantics follow the reference's distributed protocol (dist.hpp:617-800): every rank
projects its own block with the factor rows it owns, the partial sketches Z_n^g and the
partial cores G^g are summed over ranks, and the (tiny) QR is replicated on every rank so
no factor broadcast is needed. Omega and the initial factors are regenerated from the
shared seed on every rank and never communicated (paper §IV-B, dist.hpp:525-537).
"""
from __future__ import annotations

import ctypes as C

from . import _lib


def plan_slabs(dim: int, world: int):
    """Contiguous segments of `dim` over `world` ranks, lengths differing by at most one,
    longer segments first (e.g. 300 over 8 -> 38,38,38,38,37,37,37,37); the split lists
    the reference's partition() accepts (dist.hpp:70-90). Returns [(offset, length)]."""
    if world < 1 or dim < world:
        raise _lib.TenkitError("tenkit: partition: segment lengths must be positive")
    base, extra = divmod(dim, world)
    out, off = [], 0
    for r in range(world):
        ln = base + (1 if r < extra else 0)
        out.append((off, ln))
        off += ln
    return out


class DistComm:
    """Reduction hook handed to the library: `xbuf` is a device (or, in CPU tests, host)
    float64 buffer; the library writes `count` values and calls back for an all-reduce sum
    over the process group."""

    def __init__(self, slab_offset: int, global_last_dim: int, capacity: int, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.slab_offset = int(slab_offset)
        self.global_last_dim = int(global_last_dim)
        dev = device if device is not None else ("cuda" if torch.cuda.is_available() else "cpu")
        self.xbuf = torch.zeros(int(capacity), dtype=torch.float64, device=dev)
        self.calls = 0
        self._cb = _lib.ALLREDUCE_FN(self._allreduce)

    def _allreduce(self, user, count, stream) -> int:
        try:
            import torch
            import torch.distributed as dist
            if self.world > 1:
                if self.xbuf.is_cuda:
                    # enqueue on the library's stream (the one that produced xbuf and will
                    # consume the sum); NULL is the legacy default stream
                    st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
                    with torch.cuda.stream(st):
                        dist.all_reduce(self.xbuf[: int(count)], group=self.group)
                else:
                    dist.all_reduce(self.xbuf[: int(count)], group=self.group)
            self.calls += 1
            return 0
        except Exception:  # the library turns a non-zero status into "comm: allreduce failed"
            return 1

    def allreduce(self, count: int) -> int:
        return self._allreduce(None, count, None)

    def as_struct(self) -> _lib.tk_comm:
        s = _lib.tk_comm()
        s.rank = self.rank
        s.world = self.world
        s.slab_offset = self.slab_offset
        s.global_last_dim = self.global_last_dim
        s.xbuf = C.cast(C.c_void_p(self.xbuf.data_ptr()), _lib.PD)
        s.xbuf_capacity = self.xbuf.numel()
        s.allreduce_sum = self._cb
        s.user = None
        return s


def exchange_capacity(dims, ranks, oversample) -> int:
    """Doubles the reduction buffer must hold: max(I_n * r~_n, prod r~_n)."""
    rts = [min(int(r) + int(oversample), int(i)) for r, i in zip(ranks, dims)]
    core = 1
    for r in rts:
        core *= r
    return max([int(i) * r for i, r in zip(dims, rts)] + [core])


def dist_rand_tucker_2i(local_y, global_last_dim: int, slab_offset: int, ranks, oversample, seed, *, context=None,
                        group=None, **kw):
    """rand_tucker_2i of the global tensor whose last-mode slab
    [slab_offset, slab_offset + local_y.shape[-1]) lives on this rank (one process per GPU).
    Every rank returns the same model (replicated QR)."""
    from .tenkit import Context, rand_tucker_2i
    ctx = context or Context.default()
    gdims = list(local_y.shape)
    gdims[-1] = global_last_dim
    comm = DistComm(slab_offset, global_last_dim, exchange_capacity(gdims, ranks, oversample), group=group)
    ctx.set_comm(comm)
    try:
        return rand_tucker_2i(local_y, ranks, oversample, seed, context=ctx, global_last_dim=global_last_dim, **kw)
    finally:
        ctx.set_comm(None)


def dist_rand_tucker(local_y, global_last_dim: int, slab_offset: int, ranks, oversample, seed, *, context=None,
                     group=None, **kw):
    """rand_tucker (Alg. 2, tucker.hpp:108-130) of the global tensor whose last-mode slab
    lives on this rank: the Omega rows of each unfolding are drawn at their global column ids
    (dist.hpp:525-537), partial sketches and the partial core are summed over ranks, the QR
    is replicated. Every rank returns the same model."""
    from .tenkit import Context, rand_tucker
    ctx = context or Context.default()
    gdims = list(local_y.shape)
    gdims[-1] = global_last_dim
    comm = DistComm(slab_offset, global_last_dim, exchange_capacity(gdims, ranks, oversample), group=group)
    ctx.set_comm(comm)
    try:
        return rand_tucker(local_y, ranks, oversample, seed, context=ctx, global_last_dim=global_last_dim, **kw)
    finally:
        ctx.set_comm(None)
