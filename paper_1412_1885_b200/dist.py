"""Multi-GPU plumbing: block partition of Y (BlockGrid, dist.hpp:24-123; a slab of the last
mode is the 1 x ... x 1 x W grid) and the cross-rank reduction hook of the C-ABI (tk_comm),
over torch.distributed (NCCL on B200s, gloo on CPU tests).

Semantics follow the reference's distributed protocol (dist.hpp:617-800): every rank
projects its own block with the factor rows it owns, the partial sketches Z_n^g and the
partial cores G^g are summed over ranks, and the (tiny) QR is replicated on every rank so
no factor broadcast is needed. Omega and the initial factors are regenerated from the
shared seed on every rank and never communicated (paper §IV-B, dist.hpp:525-537).
"""
from __future__ import annotations

import collections
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


def ind2sub(grid_shape, w: int):
    """Column-major 1-based subscripts of worker w (dist.hpp:45-56)."""
    total = 1
    for g in grid_shape:
        total *= int(g)
    if not 1 <= w <= total:
        raise _lib.TenkitError("tenkit: ind2sub: worker id out of range")
    subs, rem = [], w - 1
    for g in grid_shape:
        subs.append(rem % int(g) + 1)
        rem //= int(g)
    return subs


def sub2ind(grid_shape, subs) -> int:
    """Inverse of ind2sub (dist.hpp:58-67)."""
    if len(subs) != len(grid_shape):
        raise _lib.TenkitError("tenkit: sub2ind: order mismatch")
    idx, stride = 0, 1
    for g, s in zip(grid_shape, subs):
        if not 1 <= s <= g:
            raise _lib.TenkitError("tenkit: sub2ind: subscript range")
        idx += (s - 1) * stride
        stride *= int(g)
    return idx + 1


class GridPlan:
    """Block partition of a tensor of `shape` into contiguous-range blocks (partition,
    dist.hpp:71-123): `splits[n]` are the segment lengths of mode n (summing to shape[n]),
    block (s_1..s_N) belongs to worker sub2ind(grid_shape, s) = rank + 1."""

    def __init__(self, shape, splits):
        self.shape = [int(d) for d in shape]
        if len(splits) != len(self.shape):
            raise _lib.TenkitError("tenkit: partition: one split list per mode required")
        self.splits, self.offsets = [], []
        for n, sp in enumerate(splits):
            sp = [int(x) for x in sp]
            if not sp:
                raise _lib.TenkitError("tenkit: partition: empty split list")
            if any(x < 1 for x in sp):
                raise _lib.TenkitError("tenkit: partition: segment lengths must be positive")
            if sum(sp) != self.shape[n]:
                raise _lib.TenkitError("tenkit: partition: split lengths must sum to the mode dimension")
            offs, o = [], 0
            for x in sp:
                offs.append(o)
                o += x
            self.splits.append(sp)
            self.offsets.append(offs)
        self.grid_shape = [len(sp) for sp in self.splits]

    @classmethod
    def even(cls, shape, grid_shape):
        """Near-even segments per mode (plan_slabs per mode)."""
        return cls(shape, [[ln for _, ln in plan_slabs(d, g)] for d, g in zip(shape, grid_shape)])

    @property
    def world(self) -> int:
        w = 1
        for g in self.grid_shape:
            w *= g
        return w

    def block(self, rank: int):
        """(lo, len) per mode of the block of 0-based `rank` (worker rank + 1)."""
        subs = ind2sub(self.grid_shape, rank + 1)
        lo = [self.offsets[n][s - 1] for n, s in enumerate(subs)]
        ln = [self.splits[n][s - 1] for n, s in enumerate(subs)]
        return lo, ln

    def local(self, y, rank: int):
        """This rank's block of a full (host) array, Fortran-ordered copy."""
        import numpy as np
        lo, ln = self.block(rank)
        return np.asfortranarray(y[tuple(slice(a, a + b) for a, b in zip(lo, ln))])


def default_grid(order: int, world: int):
    """Grid shape for `world` ranks: a slab of the last mode, except 8 ranks on a 3-way tensor,
    which get the 2 x 2 x 2 block grid (BASELINE cfg 5)."""
    if order == 3 and world == 8:
        return [2, 2, 2]
    return [1] * (order - 1) + [world]


class MessageLog:
    """Audit log of the exchanges a distributed decomposition made — the reference's
    MessageLog (dist.hpp:277-320): records in delivery order with monotone sequence numbers,
    count(kind[, mode]) and one-JSON-object-per-line output (write_ndjson).

    The B200 protocol's exchanges are all-reduces (no client, no leaders): one
    "partial_product" record (tag "z", rows = I_n, cols = r~_n) per range step and one
    "core_block" record (tag "core", rows = core elements, cols = 1) per call, each with
    source = this rank's 1-based worker id and dest = -1 (every rank). The reference's
    seed_broadcast / factor_block messages have no counterpart: the seed and Omega are
    regenerated on every rank and the basis is computed redundantly (replicated QR / Gram-eig)."""

    KINDS = ("partial_product", "seed_broadcast", "factor_block", "core_block")

    Record = collections.namedtuple("Record", "seq kind source dest mode tag rows cols")

    def __init__(self):
        self._records = []

    def append(self, kind: str, source: int, dest: int, mode: int, tag: str, rows: int, cols: int):
        if kind not in self.KINDS:
            raise _lib.TenkitError(f"tenkit: message log: unknown kind {kind}")
        self._records.append(MessageLog.Record(len(self._records), kind, int(source), int(dest), int(mode), tag,
                                               int(rows), int(cols)))

    def records(self):
        return list(self._records)

    def count(self, kind: str, mode: int | None = None) -> int:
        return sum(1 for r in self._records if r.kind == kind and (mode is None or r.mode == mode))

    def write_ndjson(self, f):
        import json
        for r in self._records:
            f.write(json.dumps(r._asdict(), separators=(",", ":")) + "\n")


def exchange_plan(alg: str, gdims, ranks, oversample):
    """The (kind, tag, mode, rows) sequence of the all-reduces one distributed call makes:
    2N range steps (Alg. 3, modes 0..N-1 twice) or N (Alg. 2), then the core."""
    order = len(gdims)
    modes = list(range(order)) * (2 if alg == "2i" else 1)
    return [("partial_product", "z", n, int(gdims[n])) for n in modes] + [("core_block", "core", -1, 0)]


class DistComm:
    """Reduction hook handed to the library: `xbuf` is a device (or, in CPU tests, host)
    float64 buffer; the library writes `count` values and calls back for an all-reduce sum
    over the process group. The block this rank holds is either a last-mode slab
    (slab_offset, global_last_dim) or, with `block_lo`/`global_dims`, a general block."""

    def __init__(self, slab_offset: int, global_last_dim: int, capacity: int, group=None, device=None,
                 block_lo=None, global_dims=None, native: bool = False):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.slab_offset = int(slab_offset)
        self.global_last_dim = int(global_last_dim)
        self.block_lo = None if block_lo is None else [int(x) for x in block_lo]
        self.global_dims = None if global_dims is None else [int(x) for x in global_dims]
        if (self.block_lo is None) != (self.global_dims is None):
            raise _lib.TenkitError("tenkit: comm: block_lo and global_dims go together")
        if self.global_dims is not None and len(self.global_dims) > _lib.TK_MAX_ORDER:
            raise _lib.TenkitError("tenkit: comm: order too large")
        dev = device if device is not None else ("cuda" if torch.cuda.is_available() else "cpu")
        self.xbuf = torch.zeros(int(capacity), dtype=torch.float64, device=dev)
        self.calls = 0
        self.log = None  # MessageLog to record into, with self.plan (exchange_plan)
        self.plan = None
        self._cb = _lib.ALLREDUCE_FN(self._allreduce)
        # native: the library's own NCCL communicator (tk_context_set_nccl) sums in place on its
        # stream — only over an NCCL process group (one process per GPU); the torch.distributed
        # callback remains for gloo (CPU tests, ranks sharing a GPU)
        self.native = bool(native) and self.world > 1 and dev != "cpu" and dist.get_backend(group) == "nccl"
        self.nccl_id = None
        if self.native:
            ids = [_lib.nccl_unique_id() if self.rank == 0 else None]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(ids, src=src, group=group)
            self.nccl_id = ids[0]

    def describe(self) -> str:
        if self.native:
            v = _lib.load().tk_nccl_version()
            return f"native NCCL {v // 10000}.{(v // 100) % 100}.{v % 100} communicator, rank {self.rank} of {self.world}"
        return f"torch.distributed callback, rank {self.rank} of {self.world}"

    def _record(self, count: int):
        if self.log is None or not self.plan:
            return
        kind, tag, mode, rows = self.plan[self.calls % len(self.plan)]
        if rows <= 0 or count % rows:
            rows = count
        self.log.append(kind, self.rank + 1, -1, mode, tag, rows, count // rows)

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
            self._record(int(count))
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
        s.allreduce_sum = self._cb  # unused with a native communicator (the library sums in place)
        s.user = None
        s.blocked = 0 if self.block_lo is None else 1
        if self.block_lo is not None:
            for n, (a, g) in enumerate(zip(self.block_lo, self.global_dims)):
                s.block_lo[n] = a
                s.global_dims[n] = g
        return s


def exchange_capacity(dims, ranks, oversample) -> int:
    """Doubles the reduction buffer must hold: max(I_n * r~_n, prod r~_n)."""
    rts = [min(int(r) + int(oversample), int(i)) for r, i in zip(ranks, dims)]
    core = 1
    for r in rts:
        core *= r
    return max([int(i) * r for i, r in zip(dims, rts)] + [core])


def _block_args(local_y, global_dims, lo):
    """(global dims, block lo) from either the slab form (int last-mode size, int offset) or
    the block form (sequences)."""
    shape = list(local_y.shape)
    if isinstance(global_dims, (int,)) or hasattr(global_dims, "__index__"):
        g = shape[:-1] + [int(global_dims)]
        l = [0] * (len(shape) - 1) + [int(lo)]
    else:
        g, l = [int(x) for x in global_dims], [int(x) for x in lo]
        if len(g) != len(shape) or len(l) != len(shape):
            raise _lib.TenkitError("tenkit: comm: one global extent and block offset per mode required")
    return g, l


def _dist_call(fn, local_y, global_dims, lo, ranks, oversample, seed, context, group, kw, alg):
    from .tenkit import Context
    ctx = context or Context.default()
    gdims, blo = _block_args(local_y, global_dims, lo)
    comm = DistComm(blo[-1], gdims[-1], exchange_capacity(gdims, ranks, oversample), group=group,
                    block_lo=blo, global_dims=gdims)
    log = kw.pop("log", None)
    if log is not None:
        comm.log = log
        comm.plan = exchange_plan(alg, gdims, ranks, oversample)
    ctx.set_comm(comm)
    try:
        return fn(local_y, ranks, oversample, seed, context=ctx, global_dims=gdims, **kw)
    finally:
        ctx.set_comm(None)


def dist_rand_tucker_2i(local_y, global_dims, lo, ranks, oversample, seed, *, context=None, group=None, **kw):
    """rand_tucker_2i (dist_rand_tucker_2i semantics, dist.hpp:884-936) of the global tensor
    whose block lives on this rank (one process per GPU): `global_dims`/`lo` are the global
    extents and the block's first index per mode (GridPlan.block), or — the slab form — the
    global last-mode size and the slab offset. Every rank returns the same model (replicated
    QR; the factors equal the single-node rand_tucker_2i's, not a rotation of them).

    DIVERGENCE FROM THE REFERENCE'S DEFAULT: the reference's dist_rand_tucker_2i orthonormalises
    with the Gram-eig transform and applies no sign rule (dist.hpp:688-723), so its factors
    match the single-node ones only up to rotation (test_dist.cpp:141-152). This default
    (orthonormalizer='colpiv') returns the single-node model (SURVEY §8e parity target);
    pass orthonormalizer='gram' for the reference's dist numerics bit-for-bit in protocol.
    log=MessageLog(): records this rank's exchanges (dist.hpp:277-320)."""
    from .tenkit import rand_tucker_2i
    return _dist_call(rand_tucker_2i, local_y, global_dims, lo, ranks, oversample, seed, context, group, kw, "2i")


def dist_rand_tucker(local_y, global_dims, lo, ranks, oversample, seed, *, context=None, group=None, **kw):
    """rand_tucker (Alg. 2, tucker.hpp:108-130; dist_rand_tucker, dist.hpp:852-878) of the
    global tensor whose block lives on this rank: the Omega rows of each unfolding are drawn
    at their global column ids (dist.hpp:496-596), partial sketches and the partial core are
    summed over ranks, the QR is replicated. Every rank returns the same model.
    Default basis 'colpiv' = single-node semantics; orthonormalizer='gram' = the reference's
    dist_rand_tucker numerics (see dist_rand_tucker_2i for the divergence note).
    log=MessageLog(): as dist_rand_tucker_2i."""
    from .tenkit import rand_tucker
    return _dist_call(rand_tucker, local_y, global_dims, lo, ranks, oversample, seed, context, group, kw, "alg2")


def dist_multiply(local_y, global_dims, lo, mode: int, r_tilde: int, seed, *, grid: GridPlan | None = None,
                  context=None, group=None):
    """dist_multiply (dist.hpp:812-846): unfold(Y, mode) * Omega with Omega =
    gaussian_matrix(prod_{k != mode} I_k, r_tilde, seed) for the global tensor Y whose block
    `local_y` (a device DenseTensor) this rank holds at offsets `lo` (GridPlan.block). Each rank
    multiplies its block's unfolding by the Omega rows of its global column ids and the partial
    products are summed over ranks (NCCL / gloo). Returns the reference's result: the Z row
    blocks, one per mode-`mode` segment of `grid` (a single block without a grid), as numpy."""
    import numpy as np
    import torch
    from .tenkit import Context, SeedSpec, _dptr, _dtype_code, _i64arr, _ptr
    ctx = context or Context.default()
    ctx.bind_torch_stream()
    seed = seed if isinstance(seed, SeedSpec) else SeedSpec(*seed)
    gdims, blo = _block_args(local_y, global_dims, lo)
    if not 0 <= mode < len(gdims):
        raise _lib.TenkitError("tenkit: dist_multiply: mode out of range")
    rows = gdims[mode]
    z = torch.empty(rows * max(int(r_tilde), 1), dtype=torch.float64, device="cuda")
    comm = DistComm(blo[-1], gdims[-1], rows * max(int(r_tilde), 1), group=group, block_lo=blo, global_dims=gdims)
    ctx.set_comm(comm)
    try:
        _lib.check(ctx.lib.tk_dist_multiply(ctx.handle, _dtype_code(local_y.data), len(gdims),
                                            _i64arr(local_y.shape), _ptr(local_y.data), int(mode), int(r_tilde),
                                            seed.root, seed.stream, _dptr(z)))
    finally:
        ctx.set_comm(None)
    zz = z.cpu().numpy().reshape((rows, int(r_tilde)), order="F")
    if grid is None:
        return [zz]
    return [zz[o:o + l] for o, l in zip(grid.offsets[mode], grid.splits[mode])]
