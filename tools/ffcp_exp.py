import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1412_1885_b200 as P
torch.manual_seed(0)
cs, I, R = 30, 1000, 20
core = torch.randn(cs ** 3, dtype=torch.float64, device="cuda")
us = [torch.linalg.qr(torch.randn(I, cs, dtype=torch.float64, device="cuda"))[0].t().contiguous().view(-1) for _ in range(3)]
m = P.TuckerModel(core, us, (cs, cs, cs))
os.environ["TENKIT_FFCP_PROF"] = "1"
for kind in (1, 0, 2):
    P.ffcp(m, R, P.ConstraintSpec(kind, 0.01), P.StopRule(200, 0.0), (1, 0))
