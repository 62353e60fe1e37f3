"""Times the cluster QR (tk_orthonormal_basis path) on Z shapes of the configs."""
import sys, os, time, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1412_1885_b200 as P
from paper_1412_1885_b200 import _lib, tenkit
ctx = tenkit._ctx(None)
import ctypes as C
for rows, cols in [(200, 15), (1000, 30), (300, 20), (2400, 40), (4000, 60)]:
    z = torch.randn(rows * cols, dtype=torch.float64, device="cuda")
    q = torch.empty(rows * cols, dtype=torch.float64, device="cuda")
    rank = C.c_int64()
    for _ in range(3):
        ctx.lib.tk_orthonormal_basis(ctx.handle, rows, cols, tenkit._dptr(z), tenkit._dptr(q), C.byref(rank), None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        ctx.lib.tk_orthonormal_basis(ctx.handle, rows, cols, tenkit._dptr(z), tenkit._dptr(q), C.byref(rank), None)
    e1.record(); torch.cuda.synchronize()
    print(f"qr {rows}x{cols}: {e0.elapsed_time(e1)/n*1000:.1f} us/call (incl. rank readback)", flush=True)
# the distributed protocol's Gram-eig basis (gram.cu) on the same shapes
for rows, cols in [(200, 15), (1000, 30), (300, 20), (2400, 40), (4000, 60)]:
    z = torch.randn(rows * cols, dtype=torch.float64, device="cuda")
    u = torch.empty(rows * cols, dtype=torch.float64, device="cuda")
    sp = torch.empty(cols, dtype=torch.float64, device="cuda")
    kept = C.c_int64()
    for _ in range(3):
        ctx.lib.tk_gram_orthonormalize(ctx.handle, rows, cols, tenkit._dptr(z), tenkit._dptr(u), tenkit._dptr(sp), C.byref(kept))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        ctx.lib.tk_gram_orthonormalize(ctx.handle, rows, cols, tenkit._dptr(z), tenkit._dptr(u), tenkit._dptr(sp), C.byref(kept))
    e1.record(); torch.cuda.synchronize()
    print(f"gram {rows}x{cols}: {e0.elapsed_time(e1)/n*1000:.1f} us/call (incl. kept readback), kept {kept.value}", flush=True)
