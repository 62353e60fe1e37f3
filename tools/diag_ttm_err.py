"""Relative error of the TTM paths (tcgen05 3xTF32 vs FFMA) against fp64, by shape and mode."""
import os, sys
import numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1412_1885_b200 as P
from oracle import pyoracle as O
O.build(); O.set_threads(os.cpu_count())
ctx = P.Context.default()
rng = np.random.default_rng(0)
for shape, mode in [((1000, 1000, 40), 1), ((1000, 1000, 40), 0), ((1000, 40, 1000), 0), ((1000, 1000, 40), 2)]:
    t = rng.standard_normal(shape).astype(np.float32)
    m = rng.standard_normal((30, shape[mode]))
    m /= np.linalg.norm(m, axis=1, keepdims=True)
    ref = O.ttm(t.astype(np.float64), m, mode)
    out = {}
    for path in ("ffma", "tc"):
        ctx.set_ttm_path(path)
        got = np.asarray(P.ttm(P.DenseTensor.from_numpy(t, np.float32), m, mode), dtype=np.float64)
        out[path] = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    print(shape, mode, {k: f"{v:.3e}" for k, v in out.items()}, flush=True)
ctx.set_ttm_path("auto")
