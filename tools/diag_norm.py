import sys, os, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_1412_1885_b200 import generators as G
y = G.generate(dict(dims=(1000,1000,1000), gen="tucker", mlrank=(20,20,20), snr=20.0))
y32 = y.float()
print("sum(y*y) fp64", float((y*y).sum()))
print("vector_norm(y)^2", float(torch.linalg.vector_norm(y))**2)
print("vector_norm(y32.double())^2", float(torch.linalg.vector_norm(y32.double()))**2)
print("vector_norm(y32)^2", float(torch.linalg.vector_norm(y32))**2)
yh = y32.double().cpu().numpy()
print("np.dot", float(np.dot(yh, yh)), "np.sum sq", float(np.sum(yh*yh)))
