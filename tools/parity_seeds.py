"""Full-size oracle parity at other seeds than the tests' seed 0: one decomposition per (config, seed)
against the streamed oracle (all r~ columns, aligned core, fit, decision margins), one JSON line each.
python tools/parity_seeds.py cfg3 1 2 3   [TENKIT_PARITY_LOG=path.jsonl]
Test infrastructure use of oracle/ (a checker), not part of the product."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1412_1885_b200 as P  # noqa: E402
from helpers import subspace_dist  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_1412_1885_b200.generators import bench_seeds, generate_as  # noqa: E402

O.build()
name = sys.argv[1]
for seed in [int(a) for a in sys.argv[2:]]:
    cfg = dict(bench.CONFIGS[name], seed=seed)
    dims = [int(d) for d in cfg["dims"]]
    y = generate_as(cfg, torch.float32)
    yd = P.DenseTensor(dims, y)
    _, alg = bench_seeds(seed)
    ranks, p = list(cfg["ranks"]), int(cfg["p"])
    m = P.rand_tucker_2i(yd, ranks, p, alg, sync_ranks=False, out="device").to_host()
    yh = y.cpu().numpy()
    del y, yd
    torch.cuda.empty_cache()
    O.set_threads(os.cpu_count() or 1)
    t0 = time.perf_counter()
    g_ref, u_ref, margins = O.rand_tucker_2i_streamed(yh, dims, ranks, p, (alg.root, alg.stream))
    t_oracle = time.perf_counter() - t0
    ysq = 0.0
    for c0 in range(0, yh.size, 1 << 27):
        c = yh[c0:c0 + (1 << 27)].astype(np.float64)
        ysq += float(np.dot(c, c))
    del yh
    sub = [subspace_dist(u, v) for u, v in zip(m.factors, u_ref)]
    aligned = O.ttm_all(m.core, [u.T @ v for u, v in zip(m.factors, u_ref)], -1, False)
    core_err = float(np.linalg.norm(aligned - g_ref) / np.linalg.norm(g_ref))
    fit = lambda g: 1.0 - float(np.sqrt(max(0.0, 1.0 - float(np.sum(np.square(g))) / ysq)))  # noqa: E731
    rec = {"tool": "parity_seeds", "config": name, "seed": seed, "subspace_all_cols": sub, "core_rel": core_err,
           "fit": fit(m.core), "fit_oracle": fit(g_ref), "pivot_margin_min": float(margins[:, 0].min()),
           "sign_margin_min": float(margins[:, 1].min()),
           "device_pivot_margin_min": float(min(m.stats["pivot_margin"])),
           "device_sign_margin_min": float(min(m.stats["sign_margin"])), "oracle_s": round(t_oracle, 1)}
    print(json.dumps(rec), flush=True)
    if os.environ.get("TENKIT_PARITY_LOG"):
        with open(os.environ["TENKIT_PARITY_LOG"], "a") as f:
            f.write(json.dumps(rec) + "\n")
