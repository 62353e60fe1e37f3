"""Python mirror of the reference `tenkit` API for the randomized-Tucker hot path.

Same names, argument meaning and error behaviour as the reference's C++ free functions
(namespace tenkit), backed by the B200 kernels through the C-ABI:

    rand_tucker_2i(y, ranks, oversample, seed)   tucker.hpp:136-169   (Alg. 3, primary)
    rand_tucker(y, ranks, oversample, seed)      tucker.hpp:108-130   (Alg. 2)
    ttm(t, m, mode)                              tensor.hpp:151-176
    ttm_all(t, ms, skip, transpose=True)         tensor.hpp:181-192
    unfold_times(t, mode, b)                     tensor.hpp:195-209
    orthonormal_basis(z)  (+ fix_column_signs)   range_finder.hpp:18-29, tucker.hpp:39-45
    gaussian_matrix(rows, cols, seed)            random.hpp:85-100
    ffcp(model, rank, constraint, stop, seed)    ffcp.hpp:94-194
    SeedSpec(root, stream).derived(...)          random.hpp:29-44

Tensors are column-major (first index fastest, tensor.hpp:31). Host inputs are numpy
arrays (any memory order; the column-major element order is what counts), device inputs
are DenseTensor objects wrapping a flat CUDA torch tensor. Invalid arguments raise
TenkitError (a ValueError) with the reference's "tenkit: ..." message.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import TenkitError, TenkitCudaError  # noqa: F401

__all__ = ["SeedSpec", "DenseTensor", "TuckerModel", "StopRule", "ConstraintSpec", "ConstraintKind", "Context",
           "rand_tucker_2i", "rand_tucker", "ttm", "ttm_all", "unfold_times", "orthonormal_basis",
           "gram_orthonormalize", "gram_ortho_transform",
           "gaussian_matrix", "ffcp", "CpModel", "model_fit", "TenkitError"]


# ---------------------------------------------------------------------------- seeds
def _mix64(x: int) -> int:
    m = (1 << 64) - 1
    x = (x + 0x9E3779B97F4A7C15) & m
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & m
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & m
    return x ^ (x >> 31)


def _hash_combine(a: int, b: int) -> int:
    m = (1 << 64) - 1
    return _mix64(a ^ ((_mix64(b) + 0x9E3779B97F4A7C15 + ((a << 6) & m) + (a >> 2)) & m))


@dataclass(frozen=True)
class SeedSpec:
    """One reproducible random stream (random.hpp:29-44)."""
    root: int = 0
    stream: int = 0

    def with_stream(self, s: int) -> "SeedSpec":
        return SeedSpec(self.root, s)

    def derived(self, *tags: int) -> "SeedSpec":
        s = self.stream
        for t in tags:
            s = _hash_combine(s, t)
        return SeedSpec(self.root, s)

    def key(self) -> int:
        return _hash_combine(_mix64(self.root), self.stream)


@dataclass(frozen=True)
class StopRule:  # cp.hpp:38-41
    max_iters: int = 1000
    fit_tol: float = 1e-6


class ConstraintKind:  # ffcp.hpp:12
    none, nonneg_mu, nonneg_hals, sparse = 0, 1, 2, 3


@dataclass(frozen=True)
class ConstraintSpec:  # ffcp.hpp:14-17
    kind: int = ConstraintKind.none
    sparsity_c: float = 0.0


# ---------------------------------------------------------------------------- tensors
class DenseTensor:
    """Column-major N-way array (tensor.hpp:32-97): `shape` + flat `data` (numpy array on
    the host or a flat CUDA torch tensor on the device), element (i_0..i_{N-1}) at
    sum_k i_k prod_{m<k} I_m."""

    def __init__(self, shape, data):
        self.shape = tuple(int(s) for s in shape)
        if len(self.shape) < 1:
            raise TenkitError("tenkit: tensor order must be at least 1")
        if any(s < 1 for s in self.shape):
            raise TenkitError("tenkit: tensor dimensions must be positive")
        n = int(np.prod(self.shape))
        if int(data.numel() if hasattr(data, "numel") else data.size) != n:
            raise TenkitError("tenkit: tensor data length does not match shape")
        self.data = data

    @staticmethod
    def from_numpy(a, dtype=np.float64) -> "DenseTensor":
        a = np.asarray(a)
        return DenseTensor(a.shape, np.ascontiguousarray(a.astype(dtype, copy=False).ravel(order="F")))

    @property
    def on_device(self) -> bool:
        return hasattr(self.data, "is_cuda") and bool(self.data.is_cuda)

    @property
    def order(self) -> int:
        return len(self.shape)

    def dim(self, n: int) -> int:
        return self.shape[n]

    @property
    def size(self) -> int:
        return int(np.prod(self.shape))

    def numpy(self) -> np.ndarray:
        d = self.data.detach().cpu().numpy() if hasattr(self.data, "detach") else np.asarray(self.data)
        return d.reshape(self.shape, order="F")

    def cuda(self, dtype=None) -> "DenseTensor":
        import torch
        d = self.data if hasattr(self.data, "is_cuda") else torch.from_numpy(np.ascontiguousarray(self.data))
        if dtype is not None:
            d = d.to(dtype)
        return DenseTensor(self.shape, d.cuda().contiguous())


@dataclass
class TuckerModel:
    """Core tensor plus one factor per mode (tucker.hpp:14-33). Host models hold numpy
    arrays (core column-major n-d array, factors I_n x R_n); device models hold flat CUDA
    torch tensors (core) and (I_n x R_n) column-major flats (factors), see `to_host`."""
    core: object
    factors: list
    core_shape: tuple = ()
    stats: dict = field(default_factory=dict)

    def order(self) -> int:
        return len(self.factors)

    def full_shape(self):
        return tuple(int(np.shape(u)[0]) if not hasattr(u, "is_cuda") else None for u in self.factors)

    def to_host(self) -> "TuckerModel":
        if isinstance(self.core, np.ndarray):
            return self
        core = self.core.detach().cpu().numpy().reshape(self.core_shape, order="F")
        fs = []
        for u, c in zip(self.factors, self.core_shape):
            a = u.detach().cpu().numpy()
            fs.append(a.reshape((a.size // c, c), order="F"))
        return TuckerModel(core, fs, self.core_shape, self.stats)


# ---------------------------------------------------------------------------- context
def _dtype_code(x) -> int:
    if hasattr(x, "dtype") and "float32" in str(x.dtype):
        return _lib.TK_F32
    if hasattr(x, "dtype") and "float64" in str(x.dtype):
        return _lib.TK_F64
    raise TenkitError("tenkit: unsupported dtype (float32 / float64 only)")


def _ptr(x):
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    return x.ctypes.data_as(C.c_void_p)


def _dptr(x):
    return C.cast(_ptr(x), _lib.PD)


def _i64arr(xs):
    return (C.c_int64 * len(xs))(*[int(v) for v in xs])


class Context:
    """A device context of libtenkit_b200 (stream, workspace, optional comm hook)."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self.lib.tk_context_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device
        self._comm_keep = None

    @classmethod
    def default(cls, device: int | None = None) -> "Context":
        if device is None:
            try:
                import torch
                device = torch.cuda.current_device() if torch.cuda.is_available() else 0
            except Exception:
                device = 0
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def bind_torch_stream(self):
        """Run on torch's current CUDA stream (so torch events bracket our kernels)."""
        import torch
        _lib.check(self.lib.tk_context_set_stream(self.handle, C.c_void_p(torch.cuda.current_stream().cuda_stream)))

    def set_ttm_path(self, path: str):
        """'auto' (tcgen05 3xTF32 for fp32 Y passes), 'ffma', 'tc' (tcgen05 whenever supported), or
        'stream' (tk_ttm on the Y-streaming kernel, ttm_stream.cu, when the shape qualifies)."""
        code = {"auto": 0, "ffma": 1, "tc": 2, "stream": 3}[path]
        _lib.check(self.lib.tk_context_set_ttm_path(self.handle, code))

    def synchronize(self):
        _lib.check(self.lib.tk_context_synchronize(self.handle))

    def set_nccl(self, unique_id: bytes | None, rank: int = 0, world: int = 0):
        """Install a native NCCL communicator (tk_context_set_nccl; None / world 0 tears it down).
        The communicator is kept across calls (its creation is expensive)."""
        if unique_id is None or world == 0:
            _lib.check(self.lib.tk_context_set_nccl(self.handle, None, 0, 0))
            self._nccl_key = None
            return
        key = (bytes(unique_id), int(rank), int(world))
        if getattr(self, "_nccl_key", None) == key:
            return
        _lib.check(self.lib.tk_context_set_nccl(self.handle, bytes(unique_id), int(rank), int(world)))
        self._nccl_key = key

    def set_comm(self, comm):
        """Install a DistComm (paper_1412_1885_b200.dist) or None. A native DistComm also
        installs (once) its NCCL communicator on this context."""
        if comm is None:
            _lib.check(self.lib.tk_context_set_comm(self.handle, None))
            self._comm_keep = None
            return
        if getattr(comm, "native", False):
            self.set_nccl(comm.nccl_id, comm.rank, comm.world)
        elif getattr(self, "_nccl_key", None) is not None:
            self.set_nccl(None)
        st = comm.as_struct()
        _lib.check(self.lib.tk_context_set_comm(self.handle, C.byref(st)))
        self._comm_keep = (comm, st)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.tk_context_destroy(self.handle)
        except Exception:
            pass


def _ctx(context):
    """The context, bound to torch's current CUDA stream so library kernels and torch ops
    are ordered (a failure to bind is an error: a silent fallback would race)."""
    c = context or Context.default()
    c.bind_torch_stream()
    return c


def _as_dense(y) -> DenseTensor:
    if isinstance(y, DenseTensor):
        return y
    return DenseTensor.from_numpy(np.asarray(y), dtype=np.asarray(y).dtype if np.asarray(y).dtype in (np.float32, np.float64) else np.float64)


def _check_ranks(y: DenseTensor, ranks, who):
    ranks = list(ranks)
    if len(ranks) != y.order:
        raise TenkitError(f"tenkit: {who}: one rank per mode required")
    return ranks


# ---------------------------------------------------------------------------- Tucker
def _tucker_call(fn_name, y, ranks, oversample, seed, context, out, opts=None):
    y = _as_dense(y)
    ranks = _check_ranks(y, ranks, fn_name[3:])
    if oversample < 0:
        raise TenkitError(f"tenkit: {fn_name[3:]}: oversampling must be nonnegative")
    seed = seed if isinstance(seed, SeedSpec) else SeedSpec(*seed)
    ctx = _ctx(context)
    gdims = list(y.shape)
    if opts is not None and getattr(opts, "_global_dims", None):
        gdims = [int(d) for d in opts._global_dims]
    elif opts is not None and getattr(opts, "_global_last_dim", None):
        gdims[-1] = opts._global_last_dim
    rts = [max(min(int(r) + int(oversample), int(i)), 1) for r, i in zip(ranks, gdims)]
    on_dev = y.on_device if out is None else (out == "device")
    if on_dev:
        import torch
        core = torch.empty(int(np.prod(rts)), dtype=torch.float64, device="cuda")
        fbufs = [torch.empty(int(i) * rt, dtype=torch.float64, device="cuda") for i, rt in zip(gdims, rts)]
    else:
        core = np.empty(int(np.prod(rts)))
        fbufs = [np.empty(int(i) * rt) for i, rt in zip(gdims, rts)]
    o = _lib.tk_tucker_out()
    o.on_device = 1 if on_dev else 0
    o.core = _dptr(core)
    for n, b in enumerate(fbufs):
        o.factors[n] = _dptr(b)
    st = _lib.tk_tucker_stats()
    args = [ctx.handle, _dtype_code(y.data), len(y.shape), _i64arr(y.shape), _ptr(y.data), 1 if y.on_device else 0,
            _i64arr(ranks), int(oversample), int(seed.root), int(seed.stream)]
    ortho = getattr(opts, "orthonormalizer", "colpiv")
    if ortho not in _ORTHO:
        raise TenkitError("tenkit: orthonormalizer must be 'colpiv' or 'gram'")
    _lib.check(ctx.lib.tk_context_set_orthonormalizer(ctx.handle, _ORTHO[ortho]))
    try:
        if fn_name == "tk_rand_tucker_2i":
            prec = getattr(opts, "precision", "native")
            if prec not in ("native", "fp64"):
                raise TenkitError("tenkit: rand_tucker_2i: precision must be 'native' or 'fp64'")
            oo = _lib.tk_tucker_opts(int(getattr(opts, "explicit_core_pass", 0)), int(getattr(opts, "sync_ranks", 1)),
                                     int(getattr(opts, "time_kernels", 0)), int(getattr(opts, "overlap", 1)),
                                     int(getattr(opts, "one_pass_per_step", 0)), 1 if prec == "fp64" else 0)
            rc = getattr(ctx.lib, fn_name)(*args, C.byref(oo), C.byref(o), C.byref(st))
        else:
            rc = getattr(ctx.lib, fn_name)(*args, C.byref(o), C.byref(st))
    finally:
        if ortho != "colpiv":
            ctx.lib.tk_context_set_orthonormalizer(ctx.handle, 0)
    _lib.check(rc)
    cshape = tuple(int(o.core_shape[n]) for n in range(y.order))
    cols = [int(o.factor_cols[n]) for n in range(y.order)]
    csize = int(np.prod(cshape))
    nsteps = 2 * y.order if fn_name == "tk_rand_tucker_2i" else y.order
    stats = {"passes": st.passes, "kernel_launches": st.kernel_launches, "y_bytes": st.y_bytes,
             "ranks": [st.ranks[i] for i in range(2 * y.order)], "stream_launches": st.stream_launches,
             "stream_ms": st.stream_ms, "pivot_margin": [st.pivot_margin[i] for i in range(nsteps)],
             "sign_margin": [st.sign_margin[i] for i in range(nsteps)],
             "qr_path": [st.qr_path[i] for i in range(nsteps)]}
    if on_dev:
        return TuckerModel(core[:csize], [b[: int(i) * c] for b, i, c in zip(fbufs, gdims, cols)], cshape, stats)
    g = core[:csize].reshape(cshape, order="F").copy()
    fs = [b[: int(i) * c].reshape((int(i), c), order="F").copy() for b, i, c in zip(fbufs, gdims, cols)]
    return TuckerModel(g, fs, cshape, stats)


# Basis of each range step: 'colpiv' = orthonormal_basis + fix_column_signs (single-node
# semantics, range_finder.hpp:18-29, tucker.hpp:39-45); 'gram' = the reference's distributed
# protocol (dist_compress_mode, dist.hpp:688-723: Gram-eig transform, U = Z T, no sign rule).
_ORTHO = {"colpiv": 0, "gram": 1}


@dataclass
class TuckerOptions:
    explicit_core_pass: int = 0
    sync_ranks: int = 1
    _global_last_dim: int = 0
    time_kernels: int = 0
    overlap: int = 1
    _global_dims: tuple = ()
    one_pass_per_step: int = 0
    orthonormalizer: str = "colpiv"
    precision: str = "native"


def rand_tucker_2i(y, ranks, oversample: int, seed, *, explicit_core_pass: bool = False, sync_ranks: bool = True,
                   context: Context | None = None, out: str | None = None, global_last_dim: int = 0,
                   time_kernels: bool = False, overlap: bool = True, global_dims=(),
                   one_pass_per_step: bool = False, orthonormalizer: str = "colpiv",
                   precision: str = "native") -> TuckerModel:
    """Alg. 3 (tucker.hpp:136-169) on the B200. `y`: numpy array (host; copied in) or a
    device DenseTensor. Returns a host (numpy) model for host input, device otherwise,
    unless out='host'/'device'. global_dims / global_last_dim: with a comm hook installed,
    y is this rank's block of a tensor of these global extents (dist.py). one_pass_per_step:
    stream Y once per range step like the reference (default: consecutive steps share a pass).
    orthonormalizer='gram': the distributed protocol's basis (dist_rand_tucker_2i numerics).
    precision='fp64' (fp32 data): fp64 arithmetic over the fp32 values, the reference's own
    precision, for data whose pivot / sign decisions (stats 'pivot_margin' / 'sign_margin')
    are closer than the default fp32-accurate passes resolve."""
    opts = TuckerOptions(int(explicit_core_pass), int(sync_ranks), int(global_last_dim), int(time_kernels),
                         int(overlap), tuple(int(d) for d in global_dims), int(one_pass_per_step), orthonormalizer,
                         precision)
    return _tucker_call("tk_rand_tucker_2i", y, ranks, oversample, seed, context, out, opts)


def rand_tucker(y, ranks, oversample: int, seed, *, context: Context | None = None, out: str | None = None,
                global_last_dim: int = 0, global_dims=(), orthonormalizer: str = "colpiv") -> TuckerModel:
    """Alg. 2 (tucker.hpp:108-130) on the B200. global_dims / global_last_dim: with a comm
    hook installed, y is this rank's block of a tensor of these global extents (dist.py).
    orthonormalizer='gram': the distributed protocol's basis (dist_rand_tucker numerics)."""
    opts = TuckerOptions(_global_last_dim=int(global_last_dim), _global_dims=tuple(int(d) for d in global_dims),
                         orthonormalizer=orthonormalizer)
    return _tucker_call("tk_rand_tucker", y, ranks, oversample, seed, context, out, opts)


# ---------------------------------------------------------------------------- kernels
def _to_dev(x, dtype):
    import torch
    if hasattr(x, "is_cuda"):
        return x.to(dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64).ravel(order="F"))).to(dtype).cuda()


def ttm(t, m, mode: int, *, dtype=None, context=None) -> np.ndarray:
    """unfold(out, n) = M unfold(T, n) (tensor.hpp:151-176); t: numpy n-d array or DenseTensor."""
    import torch
    t = _as_dense(t)
    m = np.asarray(m, dtype=np.float64)
    if not 0 <= mode < t.order:
        raise TenkitError("tenkit: mode index out of range")
    if m.ndim != 2 or m.shape[1] != t.shape[mode]:
        raise TenkitError("tenkit: ttm: matrix columns must match mode dimension")
    tdt = dtype or (torch.float32 if _dtype_code(t.data) == _lib.TK_F32 else torch.float64)
    ctx = _ctx(context)
    td = _to_dev(t.data, tdt)
    md = _to_dev(m, tdt)
    oshape = list(t.shape)
    oshape[mode] = m.shape[0]
    out = torch.empty(int(np.prod(oshape)), dtype=tdt, device="cuda")
    _lib.check(ctx.lib.tk_ttm(ctx.handle, _dtype_code(td), t.order, _i64arr(t.shape), _ptr(td), m.shape[0], _ptr(md),
                              mode, _ptr(out)))
    return out.cpu().numpy().astype(np.float64).reshape(oshape, order="F")


def ttm_all(t, ms, skip: int = -1, transpose: bool = True, *, dtype=None, context=None) -> np.ndarray:
    """ttm_all (tensor.hpp:181-192), transposed factors (the projection form)."""
    import torch
    if not transpose:
        raise TenkitError("tenkit: ttm_all: the device path applies factors transposed")
    t = _as_dense(t)
    if len(ms) != t.order:
        raise TenkitError("tenkit: ttm_all: one matrix per mode required")
    tdt = dtype or (torch.float32 if _dtype_code(t.data) == _lib.TK_F32 else torch.float64)
    ctx = _ctx(context)
    td = _to_dev(t.data, tdt)
    mds = [_to_dev(m, torch.float64) for m in ms]
    cols = [np.shape(m)[1] for m in ms]
    arr = (_lib.PD * t.order)(*[_dptr(x) for x in mds])
    oshape = [c if n != skip else t.shape[n] for n, c in enumerate(cols)]
    out = torch.empty(int(np.prod(oshape)), dtype=tdt, device="cuda")
    _lib.check(ctx.lib.tk_ttm_all(ctx.handle, _dtype_code(td), t.order, _i64arr(t.shape), _ptr(td), arr,
                                  _i64arr(cols), skip, _ptr(out)))
    return out.cpu().numpy().astype(np.float64).reshape(oshape, order="F")


def unfold_times(t, mode: int, b, *, dtype=None, context=None) -> np.ndarray:
    """unfold(T, n) * B without materialising the unfolding (tensor.hpp:195-209)."""
    import torch
    t = _as_dense(t)
    b = np.asarray(b, dtype=np.float64)
    if not 0 <= mode < t.order:
        raise TenkitError("tenkit: mode index out of range")
    if b.shape[0] != t.size // t.shape[mode]:
        raise TenkitError("tenkit: unfold_times: B rows must match unfolding width")
    tdt = dtype or (torch.float32 if _dtype_code(t.data) == _lib.TK_F32 else torch.float64)
    ctx = _ctx(context)
    td = _to_dev(t.data, tdt)
    bd = _to_dev(b, torch.float64)
    z = torch.empty(t.shape[mode] * b.shape[1], dtype=torch.float64, device="cuda")
    _lib.check(ctx.lib.tk_unfold_times(ctx.handle, _dtype_code(td), t.order, _i64arr(t.shape), _ptr(td), mode,
                                       _dptr(bd), b.shape[1], _dptr(z)))
    return z.cpu().numpy().reshape((t.shape[mode], b.shape[1]), order="F")


def orthonormal_basis(z, *, with_diag: bool = False, with_margins: bool = False, context=None):
    """Column-pivoted QR basis with the rank cut |R_kk| > 1e-12 |R_00| (range_finder.hpp:18-29),
    sign-fixed as tucker.hpp:39-45 does for every Tucker factor. with_margins: also return
    {'pivot_margin', 'sign_margin', 'qr_path'} (0 CholeskyQR2 fast path, 1 Householder)."""
    import torch
    z = np.asarray(z, dtype=np.float64)
    if z.ndim != 2 or z.shape[0] < 1:
        raise TenkitError("tenkit: orthonormal_basis: empty input")
    rows, cols = z.shape
    ctx = _ctx(context)
    zd = _to_dev(z, torch.float64)
    q = torch.zeros(rows * max(cols, 1), dtype=torch.float64, device="cuda")
    diag = torch.zeros(max(cols, 1), dtype=torch.float64, device="cuda")
    rank = C.c_int64()
    mg = np.zeros(3)
    _lib.check(ctx.lib.tk_orthonormal_basis_ex(ctx.handle, rows, cols, _dptr(zd), _dptr(q), C.byref(rank), _dptr(diag),
                                               mg.ctypes.data_as(_lib.PD)))
    r = rank.value
    u = q.cpu().numpy()[: rows * r].reshape((rows, r), order="F")
    out = [u]
    if with_diag:
        out.append(diag.cpu().numpy()[: min(rows, cols)])
    if with_margins:
        out.append({"pivot_margin": float(mg[0]), "sign_margin": float(mg[1]), "qr_path": int(mg[2])})
    return out[0] if len(out) == 1 else tuple(out)


def gram_orthonormalize(z_blocks, *, context=None):
    """gram_orthonormalize (range_finder.hpp:48-84): the row blocks' summed Gram matrix is
    eigendecomposed on the device; returns (stacked U with orthonormal columns, spectrum
    descending). Eigenvector signs are the device eigensolver's (the reference leaves them
    to Eigen's)."""
    import torch
    blocks = [np.asarray(b, dtype=np.float64) for b in z_blocks]
    if not blocks:
        raise TenkitError("tenkit: gram_orthonormalize: no blocks")
    r = blocks[0].shape[1]
    if any(b.ndim != 2 or b.shape[1] != r for b in blocks):
        raise TenkitError("tenkit: gram_orthonormalize: column-count mismatch")
    z = np.vstack(blocks)
    rows = z.shape[0]
    ctx = _ctx(context)
    zd = _to_dev(z, torch.float64)
    u = torch.zeros(rows * max(r, 1), dtype=torch.float64, device="cuda")
    sp = torch.zeros(max(r, 1), dtype=torch.float64, device="cuda")
    kept = C.c_int64()
    _lib.check(ctx.lib.tk_gram_orthonormalize(ctx.handle, rows, r, _dptr(zd), _dptr(u), _dptr(sp), C.byref(kept)))
    k = kept.value
    return u.cpu().numpy()[: rows * k].reshape((rows, k), order="F"), sp.cpu().numpy()[:k]


def gram_ortho_transform(gram, *, context=None):
    """gram_ortho_transform (range_finder.hpp:86-105) -> (transform n x kept, spectrum)."""
    import torch
    g = np.asarray(gram, dtype=np.float64)
    if g.ndim != 2 or g.shape[0] != g.shape[1]:
        raise TenkitError("tenkit: gram_ortho_transform: square Gram matrix required")
    n = g.shape[0]
    ctx = _ctx(context)
    gd = _to_dev(g, torch.float64)
    t = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    sp = torch.zeros(n, dtype=torch.float64, device="cuda")
    kept = C.c_int64()
    _lib.check(ctx.lib.tk_gram_ortho_transform(ctx.handle, n, _dptr(gd), _dptr(t), _dptr(sp), C.byref(kept)))
    k = kept.value
    return t.cpu().numpy()[: n * k].reshape((n, k), order="F"), sp.cpu().numpy()[:k]


def gaussian_matrix(rows: int, cols: int, seed, *, context=None) -> np.ndarray:
    """i.i.d. N(0,1) matrix from the counter RNG, column-major counter order (random.hpp:85-100)."""
    import torch
    seed = seed if isinstance(seed, SeedSpec) else SeedSpec(*seed)
    ctx = _ctx(context)
    out = torch.empty(max(rows * cols, 1), dtype=torch.float64, device="cuda")
    _lib.check(ctx.lib.tk_gaussian_matrix(ctx.handle, rows, cols, seed.root, seed.stream, _dptr(out)))
    return out.cpu().numpy()[: rows * cols].reshape((rows, cols), order="F")


# ---------------------------------------------------------------------------- FFCP
@dataclass
class FfcpResult:  # ffcp.hpp:81-86
    factors: list
    fit_trace: np.ndarray
    iterations: int


def ffcp(model: TuckerModel, rank: int, constraint: ConstraintSpec = ConstraintSpec(), stop: StopRule = StopRule(),
         seed=SeedSpec(), *, context: Context | None = None, out: str = "host") -> FfcpResult:
    """CP decomposition of a Tucker-compressed tensor (ffcp.hpp:94-194), computed on the device.
    A device model (from rand_tucker_2i on device data) is used in place; a host model is
    copied in. Factors come back as numpy arrays (out='host') or CUDA tensors (out='device')."""
    seed = seed if isinstance(seed, SeedSpec) else SeedSpec(*seed)
    ctx = _ctx(context)
    order = len(model.factors)
    trace = np.empty(max(stop.max_iters, 1))
    its = C.c_int()
    if hasattr(model.core, "is_cuda") and model.core.is_cuda:
        import torch
        cshape = list(model.core_shape)
        rows = [int(u.numel()) // int(c) for u, c in zip(model.factors, cshape)]
        outs = [torch.empty(int(r) * int(rank), dtype=torch.float64, device="cuda") for r in rows]
        farr = (_lib.PD * order)(*[_dptr(u) for u in model.factors])
        oarr = (_lib.PD * order)(*[_dptr(x) for x in outs])
        _lib.check(ctx.lib.tk_ffcp_device(ctx.handle, order, _i64arr(cshape), _dptr(model.core), farr, _i64arr(rows),
                                          int(rank), int(constraint.kind), float(constraint.sparsity_c),
                                          int(stop.max_iters), float(stop.fit_tol), seed.root, seed.stream, oarr,
                                          _dptr(trace), C.byref(its)))
        fs = outs if out == "device" else [o.cpu().numpy().reshape((int(r), int(rank)), order="F")
                                             for o, r in zip(outs, rows)]
        return FfcpResult(fs, trace[: its.value].copy(), its.value)
    model = model.to_host()
    core = np.ascontiguousarray(np.asarray(model.core, dtype=np.float64).ravel(order="F"))
    cshape = np.shape(model.core) if np.ndim(model.core) == order else model.core_shape
    for n, u in enumerate(model.factors):
        if np.shape(u)[1] != cshape[n]:
            raise TenkitError("tenkit: tucker model: factor columns must match core shape")
    fs = [np.ascontiguousarray(np.asarray(u, dtype=np.float64).ravel(order="F")) for u in model.factors]
    rows = [np.shape(u)[0] for u in model.factors]
    outs = [np.empty(int(r) * max(int(rank), 1)) for r in rows]
    farr = (_lib.PD * order)(*[_dptr(x) for x in fs])
    oarr = (_lib.PD * order)(*[_dptr(x) for x in outs])
    _lib.check(ctx.lib.tk_ffcp(ctx.handle, order, _i64arr(cshape), _dptr(core), farr, _i64arr(rows), int(rank),
                               int(constraint.kind), float(constraint.sparsity_c), int(stop.max_iters),
                               float(stop.fit_tol), seed.root, seed.stream, oarr, _dptr(trace), C.byref(its)))
    return FfcpResult([o.reshape((int(r), rank), order="F") for o, r in zip(outs, rows)], trace[: its.value].copy(),
                      its.value)


# ---------------------------------------------------------------------------- fit
class CpModel:  # cp.hpp:17-30
    """CP factors A_n (I_n x R): numpy arrays or CUDA tensors (I_n x R, or flat column-major)."""

    def __init__(self, factors):
        self.factors = list(factors)

    def order(self) -> int:
        return len(self.factors)


def model_fit(y, model, *, context: Context | None = None, norms: bool = False):
    """fit(y, reconstruct(model)) (tensor.hpp:282-290 with tucker.hpp:63-66) for a TuckerModel,
    or fit(y, cp_reconstruct(model)) (cp.hpp:118-128) for a CpModel / FfcpResult / factor
    list, = 1 - ||y - yhat|| / ||y||, streamed over y on the device without forming yhat.
    norms=True also returns (||y - yhat||, ||y||)."""
    import torch
    y = _as_dense(y)
    ctx = _ctx(context)
    dt = torch.float32 if _dtype_code(y.data) == _lib.TK_F32 else torch.float64
    yd = y.data if y.on_device else torch.from_numpy(np.ascontiguousarray(y.data)).cuda()
    yd = yd.to(dt).contiguous()
    order = len(y.shape)
    if isinstance(model, TuckerModel):
        cshape = [int(c) for c in (model.core_shape if model.core_shape else np.shape(model.core))]
        core = _to_dev(model.core, torch.float64) if not hasattr(model.core, "is_cuda") else model.core.contiguous()
        fac = [_to_dev(u, torch.float64) if not hasattr(u, "is_cuda") else u.contiguous() for u in model.factors]
        rank = 0
    else:
        fs = model.factors if hasattr(model, "factors") else list(model)
        rank = int(np.shape(fs[0])[1]) if not hasattr(fs[0], "is_cuda") or fs[0].dim() == 2 else \
            int(fs[0].numel()) // int(y.shape[0])
        fac = []
        for u in fs:
            if hasattr(u, "is_cuda"):
                fac.append(u.t().contiguous().view(-1) if u.dim() == 2 else u.contiguous())  # column-major flat
            else:
                fac.append(_to_dev(u, torch.float64))
        core, cshape = None, [0] * order
    if len(fac) != order:
        raise TenkitError("tenkit: fit: one factor per mode required")
    sums = np.zeros(2)
    farr = (_lib.PD * order)(*[_dptr(u) for u in fac])
    _lib.check(ctx.lib.tk_model_fit(ctx.handle, _dtype_code(yd), order, _i64arr(y.shape), _ptr(yd), _i64arr(cshape),
                                    _dptr(core) if core is not None else None, farr, int(rank), _dptr(sums)))
    res, ny = float(np.sqrt(max(sums[0], 0.0))), float(np.sqrt(max(sums[1], 0.0)))
    if not ny > 0.0:  # tensor.hpp:285
        raise TenkitError("tenkit: fit: reference tensor has zero norm")
    f = 1.0 - res / ny
    return (f, res, ny) if norms else f
