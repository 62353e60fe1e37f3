"""cfg3 (2400^3 fp32) diagnosis: device fp32 decompositions (shared passes / one pass per step)
against the streamed oracle column by column, with the per-step QR margins, and the fp64 device
path on the same (fp32-valued) data. python tools/diag_cfg3_parity.py [cfg3]"""
import json
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1412_1885_b200 as P  # noqa: E402
from helpers import subspace_dist  # noqa: E402
from oracle import pyoracle as O  # noqa: E402
from paper_1412_1885_b200.generators import bench_seeds, generate_as  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = dict(bench.CONFIGS[name], seed=0)
dims = [int(d) for d in cfg["dims"]]
ranks, p = list(cfg["ranks"]), int(cfg["p"])
_, alg = bench_seeds(0)
y = generate_as(cfg, torch.float32)
yd = P.DenseTensor(dims, y)
res = {}
for tag, kw in (("shared", {}), ("per_step", {"one_pass_per_step": True})):
    m = P.rand_tucker_2i(yd, ranks, p, alg, sync_ranks=False, out="host", **kw)
    res[tag] = m
    print(tag, "margins pivot", np.round(m.stats["pivot_margin"], 8).tolist(), "sign",
          np.round(m.stats["sign_margin"], 8).tolist(), "qr_path", m.stats["qr_path"], flush=True)
yh = y.cpu().numpy()
del y, yd
torch.cuda.empty_cache()
O.set_threads(os.cpu_count() or 1)
g_ref, u_ref, margins = O.rand_tucker_2i_streamed(yh, dims, ranks, p, (alg.root, alg.stream))
print("oracle margins", np.round(margins, 8).tolist(), flush=True)
for tag, m in res.items():
    for n, (u, v) in enumerate(zip(m.factors, u_ref)):
        dots = np.sum(u * v, axis=0)
        bad = [(j, round(float(d), 4)) for j, d in enumerate(dots) if abs(d) < 0.999]
        print(tag, "mode", n, "subspace", f"{subspace_dist(u, v):.3e}", "lead-R", f"{subspace_dist(u[:, :ranks[n]], v[:, :ranks[n]]):.3e}",
              "cols off", bad[:12], flush=True)
# fp64 device path on the same values (chunked fp32 -> fp64 upload)
n_el = yh.size
y64 = torch.empty(n_el, dtype=torch.float64, device="cuda")
step = 1 << 28
for a in range(0, n_el, step):
    y64[a:a + step] = torch.from_numpy(yh[a:a + step]).cuda().double()
yd64 = P.DenseTensor(dims, y64)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m64 = P.rand_tucker_2i(yd64, ranks, p, alg, sync_ranks=False, out="device")
    torch.cuda.synchronize()
    print("fp64 path", f"{1e3 * (time.perf_counter() - t0):.1f} ms", "passes", m64.stats["passes"], flush=True)
mh = m64.to_host()
print("fp64 subspace vs oracle", [f"{subspace_dist(u, v):.3e}" for u, v in zip(mh.factors, u_ref)],
      "core", float(np.linalg.norm(O.ttm_all(mh.core, [u.T @ v for u, v in zip(mh.factors, u_ref)], -1, False) - g_ref)
                    / np.linalg.norm(g_ref)), flush=True)
print("fp64 margins", np.round(m64.stats["sign_margin"], 8).tolist(), flush=True)
