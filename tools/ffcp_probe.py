"""Probe FFCP on the device for (core size, rank) pairs; each in its own process (a kernel
fault poisons the context). python tools/ffcp_probe.py"""
import os, subprocess, sys
CASES = [(30, 30), (40, 33), (40, 40), (60, 33), (60, 40), (60, 50), (64, 64), (50, 50)]
if len(sys.argv) > 1:
    sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
    import numpy as np
    import paper_1412_1885_b200 as P
    c, R = int(sys.argv[1]), int(sys.argv[2])
    rng = np.random.default_rng(0)
    g = rng.standard_normal((c, c, c))
    us = [np.linalg.qr(rng.standard_normal((c + 20, c)))[0] for _ in range(3)]
    res = P.ffcp(P.TuckerModel(g, us, g.shape), R, stop=P.StopRule(20, 0.0), seed=(1, 0))
    print(f"core {c}^3 R {R}: ok, fit {res.fit_trace[-1]:.6f}", flush=True)
else:
    for c, R in CASES:
        for env in ({}, {"TENKIT_FFCP_GRAPH": "1"}):
            r = subprocess.run([sys.executable, __file__, str(c), str(R)], capture_output=True, text=True,
                               env=dict(os.environ, **env), timeout=300)
            tag = "graph" if env else "persistent"
            out = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else ("FAIL " + (r.stderr.strip().splitlines() or ["?"])[-1][:150])
            print(f"{tag:10s} core {c}^3 R {R}: {out}", flush=True)
