import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import paper_1412_1885_b200 as P
from paper_1412_1885_b200 import generators as G
from oracle import pyoracle as O
dims=(1000,1000,1000)
y64 = G.generate(dict(dims=dims, gen="tucker", mlrank=(20,20,20), snr=20.0))
print("y64 sumsq", float((y64*y64).sum()))
y32 = y64.float(); del y64
_, alg = G.bench_seeds(0)
m = P.rand_tucker_2i(P.DenseTensor(dims, y32), (20,20,20), 10, alg, sync_ranks=False, out="device")
print("device core sumsq", float((m.core**2).sum()), "y32 sumsq", float((y32.double()**2).sum()))
mh = m.to_host()
yh = y32.double().cpu().numpy()
print("np.dot", float(np.dot(yh, yh)), "host core sumsq", float(np.sum(mh.core**2)))
O.set_threads(16)
print("np.dot after set_threads(16)", float(np.dot(yh, yh)))
O.set_threads(1)
print("np.dot after set_threads(1)", float(np.dot(yh, yh)))
