import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_1412_1885_b200 import generators as G
for dims in [(240,220,200), (1000,1000,1000), (600,600,600)]:
    data, _ = G.bench_seeds(0)
    y = G.gen_tucker_device(dims, (20,20,20), data)
    Y0 = y.view(dims[2]*dims[1], dims[0])  # row-major (jk, i): column-major unfold(Y,0)^T
    g = Y0.t() @ Y0
    ev = torch.linalg.eigvalsh(g).flip(0).cpu().numpy()
    print(dims, "clean top/21st:", ev[:3], ev[19:22] / ev[0], "norm2", float((y*y).sum()))
    yn = G.add_noise_device(y, 20.0, data.derived(0xAD0))
    g = Y0.t() @ Y0
    ev2 = torch.linalg.eigvalsh(g).flip(0).cpu().numpy()
    print("  noisy energy in top20:", ev2[:20].sum()/ev2.sum(), "e21/e1", ev2[20]/ev2[0])
    del y, yn, Y0, g; torch.cuda.empty_cache()
