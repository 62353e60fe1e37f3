"""ctypes binding of libtenkit_b200.so (the C-ABI in include/tenkit_b200.h).

The shared library is built in-tree by build_ext.py. There is no CPU fallback: loading
fails loudly when the library is missing, and compute calls raise when no sm_100 device
is usable.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TENKIT_B200_LIB") or os.path.join(HERE, "lib", "libtenkit_b200.so")

TK_MAX_ORDER = 8
TK_OK, TK_ERR_INVALID, TK_ERR_CUDA, TK_ERR_NO_DEVICE, TK_ERR_INTERNAL = range(5)
TK_F32, TK_F64 = 0, 1

I64 = C.c_int64
U64 = C.c_uint64
PD = C.POINTER(C.c_double)
PI64 = C.POINTER(C.c_int64)

ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p)


class tk_comm(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("slab_offset", I64), ("global_last_dim", I64),
                ("xbuf", PD), ("xbuf_capacity", I64), ("allreduce_sum", ALLREDUCE_FN), ("user", C.c_void_p),
                ("blocked", C.c_int), ("block_lo", I64 * TK_MAX_ORDER), ("global_dims", I64 * TK_MAX_ORDER)]


class tk_tucker_out(C.Structure):
    _fields_ = [("on_device", C.c_int), ("core", PD), ("core_shape", I64 * TK_MAX_ORDER),
                ("factors", PD * TK_MAX_ORDER), ("factor_cols", I64 * TK_MAX_ORDER)]


class tk_tucker_opts(C.Structure):
    _fields_ = [("explicit_core_pass", C.c_int), ("sync_ranks", C.c_int), ("time_kernels", C.c_int),
                ("overlap", C.c_int), ("one_pass_per_step", C.c_int), ("precision", C.c_int)]


class tk_tucker_stats(C.Structure):
    _fields_ = [("passes", C.c_int), ("kernel_launches", C.c_int), ("y_bytes", C.c_double),
                ("ranks", C.c_int * (2 * TK_MAX_ORDER)), ("stream_launches", C.c_int), ("stream_ms", C.c_double),
                ("pivot_margin", C.c_double * (2 * TK_MAX_ORDER)), ("sign_margin", C.c_double * (2 * TK_MAX_ORDER)),
                ("qr_path", C.c_int * (2 * TK_MAX_ORDER))]


# name -> (restype, argtypes); the exported surface of include/tenkit_b200.h
SIGNATURES = {
    "tk_last_error": (C.c_char_p, []),
    "tk_version": (C.c_int, []),
    "tk_device_ok": (C.c_int, []),
    "tk_context_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "tk_context_destroy": (C.c_int, [C.c_void_p]),
    "tk_context_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "tk_context_set_comm": (C.c_int, [C.c_void_p, C.POINTER(tk_comm)]),
    "tk_context_synchronize": (C.c_int, [C.c_void_p]),
    "tk_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "tk_context_set_nccl": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_int]),
    "tk_nccl_version": (C.c_int, []),
    "tk_qr_max_rows": (I64, [I64]),
    "tk_context_set_ttm_path": (C.c_int, [C.c_void_p, C.c_int]),
    "tk_context_set_orthonormalizer": (C.c_int, [C.c_void_p, C.c_int]),
    "tk_gram_orthonormalize": (C.c_int, [C.c_void_p, I64, I64, PD, PD, PD, PI64]),
    "tk_gram_ortho_transform": (C.c_int, [C.c_void_p, I64, PD, PD, PD, PI64]),
    "tk_rand_tucker_2i": (C.c_int, [C.c_void_p, C.c_int, I64, PI64, C.c_void_p, C.c_int, PI64, I64, U64, U64,
                                    C.POINTER(tk_tucker_opts), C.POINTER(tk_tucker_out), C.POINTER(tk_tucker_stats)]),
    "tk_rand_tucker": (C.c_int, [C.c_void_p, C.c_int, I64, PI64, C.c_void_p, C.c_int, PI64, I64, U64, U64,
                                 C.POINTER(tk_tucker_out), C.POINTER(tk_tucker_stats)]),
    "tk_ttm": (C.c_int, [C.c_void_p, C.c_int, I64, PI64, C.c_void_p, I64, C.c_void_p, I64, C.c_void_p]),
    "tk_ttm_all": (C.c_int, [C.c_void_p, C.c_int, I64, PI64, C.c_void_p, C.POINTER(PD), PI64, I64, C.c_void_p]),
    "tk_unfold_times": (C.c_int, [C.c_void_p, C.c_int, I64, PI64, C.c_void_p, I64, PD, I64, PD]),
    "tk_orthonormal_basis": (C.c_int, [C.c_void_p, I64, I64, PD, PD, PI64, PD]),
    "tk_orthonormal_basis_ex": (C.c_int, [C.c_void_p, I64, I64, PD, PD, PI64, PD, PD]),
    "tk_gaussian_matrix": (C.c_int, [C.c_void_p, I64, I64, U64, U64, PD]),
    "tk_gaussian_fill": (C.c_int, [C.c_void_p, I64, U64, U64, U64, PD]),
    "tk_gaussian_fill_block": (C.c_int, [C.c_void_p, I64, PI64, PI64, PI64, U64, U64, PD]),
    "tk_dist_multiply": (C.c_int, [C.c_void_p, C.c_int, I64, PI64, C.c_void_p, I64, I64, U64, U64, PD]),
    "tk_model_fit": (C.c_int, [C.c_void_p, C.c_int, I64, PI64, C.c_void_p, PI64, PD, C.POINTER(PD), I64, PD]),
    "tk_seed_derived": (U64, [U64, U64, U64]),
    "tk_ffcp": (C.c_int, [C.c_void_p, I64, PI64, PD, C.POINTER(PD), PI64, I64, C.c_int, C.c_double, C.c_int,
                          C.c_double, U64, U64, C.POINTER(PD), PD, C.POINTER(C.c_int)]),
    "tk_ffcp_device": (C.c_int, [C.c_void_p, I64, PI64, PD, C.POINTER(PD), PI64, I64, C.c_int, C.c_double, C.c_int,
                                 C.c_double, U64, U64, C.POINTER(PD), PD, C.POINTER(C.c_int)]),
}

_lib = None


class TenkitError(ValueError):
    """The reference's std::invalid_argument("tenkit: ...") (tensor.hpp:20-22)."""


class TenkitCudaError(RuntimeError):
    pass


def load(build_if_missing: bool = True):
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing:
        from . import build_ext
        build_ext.build()
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libtenkit_b200.so not built ({LIB_PATH}); run paper_1412_1885_b200/build_ext.py")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


TK_NCCL_UNIQUE_ID_BYTES = 128


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 of a native communicator)."""
    buf = C.create_string_buffer(TK_NCCL_UNIQUE_ID_BYTES)
    check(load().tk_nccl_unique_id(buf))
    return buf.raw


def check(rc: int):
    if rc == TK_OK:
        return
    msg = load().tk_last_error().decode()
    if rc == TK_ERR_INVALID:
        raise TenkitError(msg)
    raise TenkitCudaError(msg or f"tenkit error {rc}")
