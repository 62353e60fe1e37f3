"""ctypes front-end of the CPU oracle (oracle/tenkit_oracle.cpp) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
import this module; the product package never does. Tensors are numpy arrays in the
reference's column-major layout (first index fastest, tensor.hpp:31): pass arrays with
order='F' (or any array; they are converted).
"""
from __future__ import annotations

import ctypes as C
import glob
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libtenkit_oracle.so")
_lib = None

D = C.POINTER(C.c_double)
I64 = C.POINTER(C.c_int64)


class OracleError(ValueError):
    """Mirrors the reference's std::invalid_argument("tenkit: ...") (tensor.hpp:20-22)."""


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def openblas_path() -> str | None:
    try:
        import numpy  # noqa: F401
        libs = os.path.join(os.path.dirname(os.path.dirname(np.__file__)), "numpy.libs")
        cands = sorted(glob.glob(os.path.join(libs, "libscipy_openblas64_*.so")))
        return cands[0] if cands else None
    except Exception:
        return None


def lib(threads: int | None = None):
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.tko_last_error.restype = C.c_char_p
        _lib.tko_mix64.restype = C.c_uint64
        _lib.tko_mix64.argtypes = [C.c_uint64]
        _lib.tko_seed_key.restype = C.c_uint64
        _lib.tko_seed_key.argtypes = [C.c_uint64, C.c_uint64]
        _lib.tko_seed_derived.restype = C.c_uint64
        _lib.tko_seed_derived.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        _lib.tko_normal_at.restype = C.c_double
        _lib.tko_normal_at.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        _lib.tko_uniform_at.restype = C.c_double
        _lib.tko_uniform_at.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        _lib.tko_blas_init.argtypes = [C.c_char_p, C.c_int]
        set_threads(threads or 1)
    elif threads is not None:
        set_threads(threads)
    return _lib


def set_threads(threads: int, use_blas: bool = True) -> bool:
    """Selects OpenBLAS (ILP64, from numpy.libs) with `threads` threads for the oracle's
    large GEMMs. Returns True when OpenBLAS was found (else a fixed-order loop is used)."""
    L = _lib if _lib is not None else lib()
    if not use_blas:
        L.tko_blas_disable()
        return False
    p = openblas_path()
    return bool(L.tko_blas_init(p.encode() if p else None, int(threads)))


def _check(rc: int):
    if rc != 0:
        msg = lib().tko_last_error().decode()
        raise OracleError(msg) if rc == 1 else RuntimeError(msg)


def _f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


def _flat(a) -> np.ndarray:
    return np.ascontiguousarray(_f64(a).ravel(order="F"))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(D)


def _i64(xs) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(xs, dtype=np.int64))


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(I64)


def _tensor(flat: np.ndarray, shape) -> np.ndarray:
    return flat.reshape(tuple(int(s) for s in shape), order="F")


# ---------------------------------------------------------------- RNG (random.hpp)
def mix64(x: int) -> int:
    return int(lib().tko_mix64(x))


def seed_key(root: int, stream: int) -> int:
    return int(lib().tko_seed_key(root, stream))


def seed_derived(root: int, stream: int, *tags: int) -> tuple[int, int]:
    for t in tags:
        stream = int(lib().tko_seed_derived(root, stream, t))
    return root, stream


def normal_at(root: int, stream: int, idx: int) -> float:
    return float(lib().tko_normal_at(root, stream, idx))


def uniform_at(root: int, stream: int, idx: int) -> float:
    return float(lib().tko_uniform_at(root, stream, idx))


def gaussian_matrix(rows: int, cols: int, seed) -> np.ndarray:
    out = np.empty(rows * cols)
    _check(lib().tko_gaussian_matrix(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed[0]),
                                     C.c_uint64(seed[1]), _ptr(out)))
    return out.reshape((rows, cols), order="F")


def gaussian_rows(total_rows: int, cols: int, seed, row_ids) -> np.ndarray:
    ids = _i64(row_ids)
    out = np.empty(len(ids) * cols)
    _check(lib().tko_gaussian_rows(C.c_int64(total_rows), C.c_int64(cols), C.c_uint64(seed[0]),
                                   C.c_uint64(seed[1]), _iptr(ids), C.c_int64(len(ids)), _ptr(out)))
    return out.reshape((len(ids), cols), order="F")


# ---------------------------------------------------------------- tensor.hpp
def unfold(t, mode: int) -> np.ndarray:
    t = _f64(t)
    shape = _i64(t.shape)
    flat = _flat(t)
    if not 0 <= mode < t.ndim:
        raise OracleError("tenkit: mode index out of range")
    rows = t.shape[mode]
    out = np.empty(t.size)
    _check(lib().tko_unfold(_iptr(shape), C.c_int64(t.ndim), _ptr(flat), C.c_int64(mode), _ptr(out)))
    return out.reshape((rows, t.size // rows), order="F")


def ttm(t, m, mode: int) -> np.ndarray:
    t = _f64(t)
    m = _f64(m)
    shape = _i64(t.shape)
    flat = _flat(t)
    mf = _flat(m)
    oshape = list(t.shape)
    oshape[mode] = m.shape[0]
    out = np.empty(int(np.prod(oshape)))
    _check(lib().tko_ttm(_iptr(shape), C.c_int64(t.ndim), _ptr(flat), C.c_int64(m.shape[0]),
                         C.c_int64(m.shape[1]), _ptr(mf), C.c_int64(mode), _ptr(out)))
    return _tensor(out, oshape)


def ttm_all(t, ms, skip: int = -1, transpose: bool = False) -> np.ndarray:
    t = _f64(t)
    shape = _i64(t.shape)
    flat = _flat(t)
    mfs = [_flat(m) for m in ms]
    rows = _i64([np.shape(m)[0] for m in ms])
    cols = _i64([np.shape(m)[1] for m in ms])
    arr = (D * len(ms))(*[_ptr(x) for x in mfs])
    oshape = list(t.shape)
    for n in range(t.ndim):
        if n != skip:
            oshape[n] = int(cols[n] if transpose else rows[n])
    out = np.empty(int(np.prod(oshape)))
    osh = np.zeros(t.ndim, dtype=np.int64)
    _check(lib().tko_ttm_all(_iptr(shape), C.c_int64(t.ndim), _ptr(flat), arr, _iptr(rows), _iptr(cols),
                             C.c_int64(skip), C.c_int(1 if transpose else 0), _ptr(out), _iptr(osh)))
    return _tensor(out, osh)


def unfold_times(t, mode: int, b) -> np.ndarray:
    t = _f64(t)
    b = _f64(b)
    shape = _i64(t.shape)
    flat = _flat(t)
    bf = _flat(b)
    out = np.empty(t.shape[mode] * b.shape[1])
    _check(lib().tko_unfold_times(_iptr(shape), C.c_int64(t.ndim), _ptr(flat), C.c_int64(mode),
                                  C.c_int64(b.shape[0]), C.c_int64(b.shape[1]), _ptr(bf), _ptr(out)))
    return out.reshape((t.shape[mode], b.shape[1]), order="F")


def fit(y, yhat) -> float:
    y = _f64(y)
    shape = _i64(y.shape)
    a, b = _flat(y), _flat(yhat)
    out = C.c_double()
    _check(lib().tko_fit(_iptr(shape), C.c_int64(y.ndim), _ptr(a), _ptr(b), C.byref(out)))
    return out.value


# ---------------------------------------------------------------- range_finder.hpp
def orthonormal_basis(z, diagnostics: bool = False):
    z = _f64(z)
    if z.ndim != 2:
        raise OracleError("tenkit: orthonormal_basis: matrix input required")
    rows, cols = z.shape
    zf = _flat(z)
    q = np.empty(rows * max(cols, 1))
    rank = C.c_int64()
    perm = np.zeros(max(cols, 1), dtype=np.int64)
    size = max(min(rows, cols), 1)
    rdiag = np.zeros(size)
    margin = np.zeros(size)
    _check(lib().tko_orthonormal_basis(C.c_int64(rows), C.c_int64(cols), _ptr(zf), _ptr(q), C.byref(rank),
                                       _iptr(perm), _ptr(rdiag), _ptr(margin)))
    r = rank.value
    u = q[: rows * r].reshape((rows, r), order="F").copy()
    if diagnostics:
        return u, {"perm": perm[:cols], "rdiag": rdiag[: min(rows, cols)], "pivot_margin": margin[: min(rows, cols)]}
    return u


def fix_column_signs(u) -> np.ndarray:
    u = _f64(u)
    f = _flat(u).copy()
    _check(lib().tko_fix_column_signs(C.c_int64(u.shape[0]), C.c_int64(u.shape[1]), _ptr(f)))
    return f.reshape(u.shape, order="F")


# ---------------------------------------------------------------- tucker.hpp
def _model_buffers(dims, ranks, p):
    rts = [min(int(r) + int(p), int(i)) for r, i in zip(ranks, dims)]
    core = np.empty(int(np.prod(rts)))
    cshape = np.zeros(len(dims), dtype=np.int64)
    fbufs = [np.empty(int(i) * rt) for i, rt in zip(dims, rts)]
    farr = (D * len(dims))(*[_ptr(b) for b in fbufs])
    cols = np.zeros(len(dims), dtype=np.int64)
    return rts, core, cshape, fbufs, farr, cols


def _unpack_model(dims, core, cshape, fbufs, cols):
    n = int(np.prod(cshape))
    g = _tensor(core[:n].copy(), cshape)
    us = [b[: int(i) * int(c)].reshape((int(i), int(c)), order="F").copy() for b, i, c in zip(fbufs, dims, cols)]
    return g, us


def rand_tucker_2i(y, ranks, oversample: int, seed, return_sketches: bool = False):
    """Alg. 3 (tucker.hpp:136-169). Returns (core, factors[, Z sketches])."""
    y = _f64(y)
    dims = y.shape
    shape = _i64(dims)
    flat = _flat(y)
    rts, core, cshape, fbufs, farr, cols = _model_buffers(dims, ranks, oversample)
    zarr = None
    zbufs = []
    if return_sketches:
        for _pass in range(2):
            for n in range(y.ndim):
                zbufs.append(np.empty(int(dims[n]) * rts[n]))
        zarr = (D * len(zbufs))(*[_ptr(b) for b in zbufs])
    _check(lib().tko_rand_tucker_2i(_iptr(shape), C.c_int64(y.ndim), _ptr(flat), _iptr(_i64(ranks)),
                                    C.c_int64(oversample), C.c_uint64(seed[0]), C.c_uint64(seed[1]),
                                    _ptr(core), _iptr(cshape), farr, _iptr(cols), zarr))
    g, us = _unpack_model(dims, core, cshape, fbufs, cols)
    if return_sketches:
        zs = [b.reshape((int(dims[i % y.ndim]), rts[i % y.ndim]), order="F") for i, b in enumerate(zbufs)]
        return g, us, zs
    return g, us


def rand_tucker_2i_streamed(y32, dims, ranks, oversample: int, seed, slab_elems: int = 1 << 25,
                            return_sketches: bool = False):
    """Alg. 3 (tucker.hpp:136-169) streamed over last-mode slabs of an fp32 host tensor
    (flat column-major np.float32 of prod(dims) elements; each slab converted to fp64):
    the full-size parity checker for tensors whose fp64 copy does not fit in host memory
    (dist.hpp:496-596 streaming pattern). Returns (core, factors, margins[, sketches]) with
    margins = per step (pivot margin, sign margin)."""
    y32 = np.ascontiguousarray(np.asarray(y32, dtype=np.float32).reshape(-1))
    dims = [int(d) for d in dims]
    if y32.size != int(np.prod(dims)):
        raise OracleError("tenkit: tensor data length does not match shape")
    order = len(dims)
    rts, core, cshape, fbufs, farr, cols = _model_buffers(dims, ranks, oversample)
    zarr, zbufs = None, []
    if return_sketches:
        zbufs = [np.empty(dims[i % order] * rts[i % order]) for i in range(2 * order)]
        zarr = (D * len(zbufs))(*[_ptr(b) for b in zbufs])
    margins = np.zeros(4 * order)
    _check(lib().tko_rand_tucker_2i_f32_streamed(
        _iptr(_i64(dims)), C.c_int64(order), y32.ctypes.data_as(C.POINTER(C.c_float)), _iptr(_i64(ranks)),
        C.c_int64(oversample), C.c_uint64(seed[0]), C.c_uint64(seed[1]), C.c_int64(slab_elems), _ptr(core),
        _iptr(cshape), farr, _iptr(cols), zarr, _ptr(margins)))
    g, us = _unpack_model(dims, core, cshape, fbufs, cols)
    mg = margins.reshape(2 * order, 2)
    if return_sketches:
        zs = [b.reshape((dims[i % order], rts[i % order]), order="F") for i, b in enumerate(zbufs)]
        return g, us, mg, zs
    return g, us, mg


def sym_eig(a):
    """Symmetric eigendecomposition (stand-in for Eigen's SelfAdjointEigenSolver,
    range_finder.hpp:57,87): ascending eigenvalues, eigenvectors as columns."""
    a = _f64(a)
    n = a.shape[0]
    ev = np.empty(max(n, 1))
    vec = np.empty(max(n * n, 1))
    _check(lib().tko_sym_eig(C.c_int64(n), _ptr(_flat(a)), _ptr(ev), _ptr(vec)))
    return ev[:n], vec[: n * n].reshape((n, n), order="F")


def gram_ortho_transform(gram):
    """gram_ortho_transform (range_finder.hpp:86-105) -> (transform n x kept, spectrum)."""
    gram = _f64(gram)
    n = gram.shape[0]
    t = np.empty(max(n * n, 1))
    sp = np.empty(max(n, 1))
    kept = C.c_int64()
    _check(lib().tko_gram_ortho_transform(C.c_int64(n), _ptr(_flat(gram)), _ptr(t), _ptr(sp), C.byref(kept)))
    k = kept.value
    return t[: n * k].reshape((n, k), order="F").copy(), sp[:k].copy()


def gram_orthonormalize(z_blocks):
    """gram_orthonormalize (range_finder.hpp:48-84) over row blocks -> (stacked U, spectrum)."""
    blocks = [_f64(b) for b in z_blocks]
    cols = blocks[0].shape[1] if blocks else 0
    z = np.vstack(blocks) if blocks else np.zeros((0, 0))
    rows = z.shape[0]
    br = _i64([b.shape[0] for b in blocks])
    u = np.empty(max(rows * cols, 1))
    sp = np.empty(max(cols, 1))
    kept = C.c_int64()
    _check(lib().tko_gram_orthonormalize(C.c_int64(len(blocks)), _iptr(br), C.c_int64(cols), _ptr(_flat(z)),
                                         _ptr(u), _ptr(sp), C.byref(kept)))
    k = kept.value
    return u[: rows * k].reshape((rows, k), order="F").copy(), sp[:k].copy()


def dist_rand_tucker_gram(y, ranks, oversample: int, seed, alg: int = 3):
    """The reference's distributed algorithms' numerics (dist_rand_tucker alg=2,
    dist_rand_tucker_2i alg=3; dist.hpp:852-936): Gram-eig basis, no sign rule,
    on the assembled tensor. Returns (core, factors)."""
    y = _f64(y)
    dims = y.shape
    rts, core, cshape, fbufs, farr, cols = _model_buffers(dims, ranks, oversample)
    _check(lib().tko_dist_rand_tucker_gram(C.c_int(alg), _iptr(_i64(dims)), C.c_int64(y.ndim), _ptr(_flat(y)),
                                           _iptr(_i64(ranks)), C.c_int64(oversample), C.c_uint64(seed[0]),
                                           C.c_uint64(seed[1]), _ptr(core), _iptr(cshape), farr, _iptr(cols)))
    return _unpack_model(dims, core, cshape, fbufs, cols)


def rand_tucker(y, ranks, oversample: int, seed):
    """Alg. 2 (tucker.hpp:108-130). Returns (core, factors)."""
    y = _f64(y)
    dims = y.shape
    shape = _i64(dims)
    flat = _flat(y)
    # Alg. 2 caps r_tilde by the *current* mode size, which equals I_n (modes are shrunk in order)
    rts, core, cshape, fbufs, farr, cols = _model_buffers(dims, ranks, oversample)
    _check(lib().tko_rand_tucker(_iptr(shape), C.c_int64(y.ndim), _ptr(flat), _iptr(_i64(ranks)),
                                 C.c_int64(oversample), C.c_uint64(seed[0]), C.c_uint64(seed[1]),
                                 _ptr(core), _iptr(cshape), farr, _iptr(cols)))
    return _unpack_model(dims, core, cshape, fbufs, cols)


def reconstruct(core, factors) -> np.ndarray:
    core = _f64(core)
    cshape = _i64(core.shape)
    cf = _flat(core)
    fs = [_flat(u) for u in factors]
    rows = _i64([np.shape(u)[0] for u in factors])
    arr = (D * len(fs))(*[_ptr(x) for x in fs])
    out = np.empty(int(np.prod(rows)))
    _check(lib().tko_reconstruct(_iptr(cshape), C.c_int64(core.ndim), _ptr(cf), arr, _iptr(rows), _ptr(out)))
    return _tensor(out, rows)


# ---------------------------------------------------------------- bench.hpp generators
def gen_tucker(dims, mlranks, seed) -> np.ndarray:
    out = np.empty(int(np.prod(dims)))
    _check(lib().tko_gen_tucker(_iptr(_i64(dims)), _iptr(_i64(mlranks)), C.c_int64(len(dims)),
                                C.c_uint64(seed[0]), C.c_uint64(seed[1]), _ptr(out)))
    return _tensor(out, dims)


CP_GAUSSIAN, CP_EXPONENTIAL, CP_UNIFORM = 0, 1, 2


def gen_cp(dims, rank: int, kind: int, seed, zero_frac: float = 0.0):
    out = np.empty(int(np.prod(dims)))
    fb = [np.empty(int(i) * rank) for i in dims]
    arr = (D * len(dims))(*[_ptr(b) for b in fb])
    _check(lib().tko_gen_cp(_iptr(_i64(dims)), C.c_int64(len(dims)), C.c_int64(rank), C.c_int(kind),
                            C.c_double(zero_frac), C.c_uint64(seed[0]), C.c_uint64(seed[1]), _ptr(out), arr))
    return _tensor(out, dims), [b.reshape((int(i), rank), order="F") for b, i in zip(fb, dims)]


def add_noise(y, snr_db: float, seed, abs_noise: bool = False) -> np.ndarray:
    y = _f64(y)
    f = _flat(y).copy()
    _check(lib().tko_add_noise(_iptr(_i64(y.shape)), C.c_int64(y.ndim), _ptr(f), C.c_double(snr_db),
                               C.c_uint64(seed[0]), C.c_uint64(seed[1]), C.c_int(1 if abs_noise else 0)))
    return _tensor(f, y.shape)


# ---------------------------------------------------------------- ffcp.hpp / cp.hpp
NONE, NONNEG_MU, NONNEG_HALS, SPARSE = 0, 1, 2, 3


def ffcp(core, factors, rank: int, constraint: int = NONE, sparsity_c: float = 0.0,
         max_iters: int = 1000, fit_tol: float = 1e-6, seed=(0, 0)):
    """ffcp (ffcp.hpp:94-194). Returns (cp_factors, fit_trace, iterations)."""
    core = _f64(core)
    cshape = _i64(core.shape)
    cf = _flat(core)
    us = [_flat(u) for u in factors]
    rows = _i64([np.shape(u)[0] for u in factors])
    uarr = (D * len(us))(*[_ptr(x) for x in us])
    ob = [np.empty(int(r) * rank) for r in rows]
    oarr = (D * len(ob))(*[_ptr(x) for x in ob])
    trace = np.empty(max(max_iters, 1))
    its = C.c_int()
    _check(lib().tko_ffcp(_iptr(cshape), C.c_int64(core.ndim), _ptr(cf), uarr, _iptr(rows), C.c_int64(rank),
                          C.c_int(constraint), C.c_double(sparsity_c), C.c_int(max_iters), C.c_double(fit_tol),
                          C.c_uint64(seed[0]), C.c_uint64(seed[1]), oarr, _ptr(trace), C.byref(its)))
    fs = [b.reshape((int(r), rank), order="F") for b, r in zip(ob, rows)]
    return fs, trace[: its.value].copy(), its.value


def cp_reconstruct(factors) -> np.ndarray:
    dims = _i64([np.shape(a)[0] for a in factors])
    rank = int(np.shape(factors[0])[1])
    fs = [_flat(a) for a in factors]
    arr = (D * len(fs))(*[_ptr(x) for x in fs])
    out = np.empty(int(np.prod(dims)))
    _check(lib().tko_cp_reconstruct(_iptr(dims), C.c_int64(len(dims)), C.c_int64(rank), arr, _ptr(out)))
    return _tensor(out, dims)


# ---------------------------------------------------------------- oracle/_ref: the reference's own code
_REF_PATH = os.path.join(_HERE, "_ref", "libtenkit_ref.so")
_ref = None


def ref_available() -> bool:
    """True where oracle/_ref was built (this container: /root/reference present)."""
    return os.path.exists(_REF_PATH)


def ref_lib():
    """The reference's hot-path headers (tensor/random/range_finder/tucker.hpp, unmodified)
    compiled against oracle/ref_shim (Eigen API over LAPACK) — fixture generation only."""
    global _ref
    if _ref is None:
        if not ref_available():
            subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)
        if not ref_available():
            raise RuntimeError("oracle/_ref not built (reference sources absent)")
        _ref = C.CDLL(_REF_PATH)
        _ref.tkr_last_error.restype = C.c_char_p
        _ref.tkr_normal_at.restype = C.c_double
        _ref.tkr_normal_at.argtypes = [C.c_uint64] * 3
        _ref.tkr_seed_derived.restype = C.c_uint64
        _ref.tkr_seed_derived.argtypes = [C.c_uint64] * 3
        p = openblas_path()
        if not p or _ref.tkr_init(p.encode()) != 0:
            raise RuntimeError("oracle/_ref: LAPACK (OpenBLAS) not found")
    return _ref


def _rcheck(rc):
    if rc != 0:
        msg = ref_lib().tkr_last_error().decode()
        raise OracleError(msg) if rc == 1 else RuntimeError(msg)


def ref_gaussian_matrix(rows: int, cols: int, seed) -> np.ndarray:
    out = np.empty(rows * cols)
    _rcheck(ref_lib().tkr_gaussian_matrix(C.c_int64(rows), C.c_int64(cols), C.c_uint64(seed[0]), C.c_uint64(seed[1]),
                                          _ptr(out)))
    return out.reshape((rows, cols), order="F")


def ref_ttm(t, m, mode: int) -> np.ndarray:
    t, m = _f64(t), _f64(m)
    oshape = list(t.shape)
    oshape[mode] = m.shape[0]
    out = np.empty(int(np.prod(oshape)))
    _rcheck(ref_lib().tkr_ttm(_iptr(_i64(t.shape)), C.c_int64(t.ndim), _ptr(_flat(t)), C.c_int64(m.shape[0]),
                              C.c_int64(m.shape[1]), _ptr(_flat(m)), C.c_int64(mode), _ptr(out)))
    return _tensor(out, oshape)


def ref_unfold_times(t, mode: int, b) -> np.ndarray:
    t, b = _f64(t), _f64(b)
    out = np.empty(t.shape[mode] * b.shape[1])
    _rcheck(ref_lib().tkr_unfold_times(_iptr(_i64(t.shape)), C.c_int64(t.ndim), _ptr(_flat(t)), C.c_int64(mode),
                                       C.c_int64(b.shape[0]), C.c_int64(b.shape[1]), _ptr(_flat(b)), _ptr(out)))
    return out.reshape((t.shape[mode], b.shape[1]), order="F")


def ref_orthonormal_basis(z) -> np.ndarray:
    """orthonormal_basis + fix_column_signs of the reference (range_finder.hpp:18-29, tucker.hpp:39-45)."""
    z = _f64(z)
    rows, cols = z.shape
    q = np.empty(rows * max(cols, 1))
    rank = C.c_int64()
    _rcheck(ref_lib().tkr_orthonormal_basis(C.c_int64(rows), C.c_int64(cols), _ptr(_flat(z)), _ptr(q), C.byref(rank)))
    return q[: rows * rank.value].reshape((rows, rank.value), order="F").copy()


def _ref_tucker(fn, y, ranks, oversample, seed):
    y = _f64(y)
    dims = y.shape
    rts, core, cshape, fbufs, farr, cols = _model_buffers(dims, ranks, oversample)
    _rcheck(fn(_iptr(_i64(dims)), C.c_int64(y.ndim), _ptr(_flat(y)), _iptr(_i64(ranks)), C.c_int64(oversample),
               C.c_uint64(seed[0]), C.c_uint64(seed[1]), _ptr(core), _iptr(cshape), farr, _iptr(cols)))
    return _unpack_model(dims, core, cshape, fbufs, cols)


def ref_rand_tucker_2i(y, ranks, oversample: int, seed):
    """The reference's rand_tucker_2i (tucker.hpp:136-169) itself. Returns (core, factors)."""
    return _ref_tucker(ref_lib().tkr_rand_tucker_2i, y, ranks, oversample, seed)


def ref_rand_tucker(y, ranks, oversample: int, seed):
    """The reference's rand_tucker (Alg. 2, tucker.hpp:108-130) itself. Returns (core, factors)."""
    return _ref_tucker(ref_lib().tkr_rand_tucker, y, ranks, oversample, seed)
