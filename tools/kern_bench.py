"""In-situ timings (CUDA events, warm caches, boost clocks) of the small kernels of a cfg-2 step:
tk_ttm on the second-stage / core shapes and the cluster QR. python tools/kern_bench.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_1412_1885_b200 import _lib, tenkit  # noqa: E402

ctx = tenkit._ctx(None)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for dims, mode, rows in [((30, 1000, 30), 1, 30), ((1000, 1000, 30), 1, 30), ((30, 1000, 1000), 1, 30),
                         ((1000, 30, 1000), 2, 30), ((1000, 1000, 30), 0, 30)]:
    t = torch.randn(int(np.prod(dims)), dtype=torch.float32, device="cuda")
    m = torch.randn(rows * dims[mode], dtype=torch.float32, device="cuda")
    od = list(dims)
    od[mode] = rows
    out = torch.empty(int(np.prod(od)), dtype=torch.float32, device="cuda")
    arr = (_lib.I64 * 3)(*dims)
    us = timeit(lambda: _lib.check(ctx.lib.tk_ttm(ctx.handle, 0, 3, arr, tenkit._ptr(t), rows, tenkit._ptr(m), mode,
                                                  tenkit._ptr(out))))
    print(f"ttm {dims} mode {mode} -> {rows}: {us:.1f} us (incl. factor pack)", flush=True)
for rows, cols in [(1000, 30), (300, 20)]:
    z = torch.randn(rows * cols, dtype=torch.float64, device="cuda")
    q = torch.empty(rows * cols, dtype=torch.float64, device="cuda")
    rank = C.c_int64()
    us = timeit(lambda: ctx.lib.tk_orthonormal_basis(ctx.handle, rows, cols, tenkit._dptr(z), tenkit._dptr(q),
                                                     C.byref(rank), None))
    print(f"qr {rows}x{cols}: {us:.1f} us/call (incl. rank read-back)", flush=True)
