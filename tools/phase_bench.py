"""Where a decomposition goes, per phase (eager run, CUDA events around every phase):
TENKIT_PHASE_TIMING=1 TENKIT_NO_GRAPH=1 python tools/phase_bench.py [cfg2|cfg3|cfg4|cfg1]"""
import os
import sys

os.environ.setdefault("TENKIT_PHASE_TIMING", "1")
os.environ.setdefault("TENKIT_NO_GRAPH", "1")
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1412_1885_b200 as P  # noqa: E402
from paper_1412_1885_b200.generators import bench_seeds, generate_as  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]
tdt = torch.float32 if cfg["dtype"] == "f32" else torch.float64
y = generate_as(dict(cfg, seed=0), tdt)
yd = P.DenseTensor(list(cfg["dims"]), y)
_, seed = bench_seeds(0)
for it in range(4):
    m = P.rand_tucker_2i(yd, cfg["ranks"], cfg["p"], seed, sync_ranks=False, out="device")
    torch.cuda.synchronize()
print("passes", m.stats["passes"], "launches", m.stats["kernel_launches"])
