"""cfg2 full size: per-mode subspace distance to the fp64 oracle for each TTM path setting."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import paper_1412_1885_b200 as P
from paper_1412_1885_b200 import generators as G
from oracle import pyoracle as O
from helpers import subspace_dist
dims, ranks, p = (1000, 1000, 1000), (20, 20, 20), 10
y64 = G.generate(dict(dims=dims, gen="tucker", mlrank=(20, 20, 20), snr=20.0))
y32 = y64.float(); del y64
_, alg = G.bench_seeds(0)
yh = y32.double().cpu().numpy()
O.build(); O.set_threads(os.cpu_count())
g_ref, u_ref = O.rand_tucker_2i(yh.reshape(dims, order="F"), ranks, p, (alg.root, alg.stream))
ctx = P.Context.default()
for path in ("auto", "ffma", "tc"):
    ctx.set_ttm_path(path)
    m = P.rand_tucker_2i(P.DenseTensor(dims, y32), ranks, p, alg, sync_ranks=False, out="device").to_host()
    d = [subspace_dist(u, v) for u, v in zip(m.factors, u_ref)]
    d20 = [subspace_dist(u[:, :20], v[:, :20]) for u, v in zip(m.factors, u_ref)]
    print(f"{path}: subspace dist {['%.3e' % x for x in d]}  leading-20 {['%.3e' % x for x in d20]}", flush=True)
ctx.set_ttm_path("auto")
