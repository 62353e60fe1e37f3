"""Times device FFCP on a config-2-sized Tucker model (core 30^3, U 1000x30, CP rank 20; or
`python tools/ffcp_bench.py iters core I R`, e.g. 200 40 2400 30 for cfg 3):
the persistent cooperative kernel (default) against the per-sweep CUDA graph
(TENKIT_FFCP_GRAPH=1), and the largest fit-trace difference between the two."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1412_1885_b200 as P
torch.manual_seed(0)
cs, I, R = (int(a) for a in sys.argv[2:5]) if len(sys.argv) >= 5 else (30, 1000, 20)
core = torch.randn(cs ** 3, dtype=torch.float64, device="cuda")
us = [torch.linalg.qr(torch.randn(I, cs, dtype=torch.float64, device="cuda"))[0].t().contiguous().view(-1) for _ in range(3)]
m = P.TuckerModel(core, us, (cs, cs, cs))
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
for kind in (0, 1, 2, 3):
    res = {}
    for path in ("graph", "persistent"):
        os.environ["TENKIT_FFCP_GRAPH"] = "1" if path == "graph" else "0"
        P.ffcp(m, R, P.ConstraintSpec(kind, 0.01), P.StopRule(5, 0.0), (1, 0))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = P.ffcp(m, R, P.ConstraintSpec(kind, 0.01), P.StopRule(iters, 0.0), (1, 0))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        res[path] = r
        print(f"ffcp kind {kind} {path}: {r.iterations} iterations in {dt*1e3:.2f} ms ({dt/r.iterations*1e6:.1f} us/iter)"
              f" final fit {r.fit_trace[-1]:.12f}", flush=True)
    d = np.max(np.abs(np.asarray(res["graph"].fit_trace) - np.asarray(res["persistent"].fit_trace)))
    print(f"  max |fit graph - persistent| = {d:.3e}", flush=True)
os.environ.pop("TENKIT_FFCP_GRAPH")
