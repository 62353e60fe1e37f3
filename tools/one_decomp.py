"""One eager decomposition of a bench config (for ncu captures of its kernels):
TENKIT_NO_GRAPH=1 python tools/one_decomp.py cfg3 [reps]"""
import os
import sys

os.environ.setdefault("TENKIT_NO_GRAPH", "1")
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1412_1885_b200 as P  # noqa: E402
from paper_1412_1885_b200.generators import bench_seeds, generate_as  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = bench.CONFIGS[name]
tdt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
y = generate_as(dict(cfg, seed=0), tdt)
torch.cuda.empty_cache()
yd = P.DenseTensor(list(cfg["dims"]), y)
_, seed = bench_seeds(0)
for it in range(reps):
    m = P.rand_tucker_2i(yd, cfg["ranks"], cfg["p"], seed, sync_ranks=False, out="device")
    torch.cuda.synchronize()
print(name, "passes", m.stats["passes"], "launches", m.stats["kernel_launches"], flush=True)
