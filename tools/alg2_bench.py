"""rand_tucker (Alg. 2) vs rand_tucker_2i (ColPiv and Gram-eig bases) at cfg 2 on device data."""
import os, sys, time
import torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1412_1885_b200 as P
from paper_1412_1885_b200.generators import generate_as, bench_seeds
dims = (1000, 1000, 1000)
y = generate_as(dict(dims=dims, gen="tucker", mlrank=(20, 20, 20), snr=20.0), torch.float32)
yd = P.DenseTensor(dims, y)
_, alg = bench_seeds(0)
ctx = P.Context.default(); ctx.bind_torch_stream()
for name, fn, kw in [("rand_tucker (Alg 2)", P.rand_tucker, {}), ("rand_tucker_2i", P.rand_tucker_2i, dict(sync_ranks=False)),
                     ("rand_tucker_2i explicit core", P.rand_tucker_2i, dict(sync_ranks=False, explicit_core_pass=True)),
                     ("rand_tucker_2i, Gram-eig basis", P.rand_tucker_2i, dict(sync_ranks=False, orthonormalizer="gram")),
                     ("rand_tucker (Alg 2), Gram-eig basis", P.rand_tucker, dict(orthonormalizer="gram"))]:
    for _ in range(3):
        m = fn(yd, (20, 20, 20), 10, alg, out="device", **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        m = fn(yd, (20, 20, 20), 10, alg, out="device", **kw)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{name}: {ms:.2f} ms/call, passes {m.stats['passes']}", flush=True)
