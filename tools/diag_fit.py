import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1412_1885_b200 as P
from paper_1412_1885_b200 import generators as G
for dims in [(240,220,200), (600,600,600), (1000,1000,1000)]:
    data, alg = G.bench_seeds(0)
    y = G.generate(dict(dims=dims, gen="tucker", mlrank=(20,20,20), snr=20.0))
    y32 = y.float()
    m = P.rand_tucker_2i(P.DenseTensor(dims, y32), (20,20,20), 10, alg, out="device").to_host()
    ysq = float((y*y).sum())
    out = []
    for n in range(3):
        yt = y.view(*reversed(dims))  # [k][j][i]
        ax = 2 - n
        U = torch.from_numpy(m.factors[n]).cuda()
        proj = torch.tensordot(yt, U, dims=([ax], [0]))
        out.append(float((proj*proj).sum())/ysq)
    print(dims, "mode captured energy", out, "core energy", float((m.core**2).sum())/ysq, "ranks", m.stats["ranks"], flush=True)
    # the same with explicit core pass and sync ranks
    m2 = P.rand_tucker_2i(P.DenseTensor(dims, y32), (20,20,20), 10, alg, out="device", explicit_core_pass=True).to_host()
    print("   explicit core energy", float((m2.core**2).sum())/ysq, flush=True)
    del y, y32, proj; torch.cuda.empty_cache()
