"""The library's native NCCL communicator (tk_nccl_unique_id / tk_context_set_nccl) on the one
GPU available: a world-1 communicator runs the same ncclAllReduce calls (in place, fp64, on the
call's stream) that an N-GPU run makes, inside the captured CUDA graph on repeated calls. The
model must equal the no-communicator model bit for bit (a 1-rank sum is the identity)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1412_1885_b200 as P
    return P


def test_native_nccl_world1_matches_no_comm(P, O):
    import torch
    from paper_1412_1885_b200 import _lib
    lib = _lib.load()
    assert lib.tk_nccl_version() >= 21800
    seed = (4, 4)
    dims = (160, 150, 140)
    y = O.add_noise(O.gen_tucker(dims, (5, 5, 5), seed), 20.0, O.seed_derived(*seed, 0xAD0)).astype(np.float32)
    yd = P.DenseTensor.from_numpy(y, np.float32).cuda()
    plain = P.Context(0)
    ref = P.rand_tucker_2i(yd, (8, 8, 8), 4, (1, 3), context=plain, sync_ranks=False, out="host")

    ctx = P.Context(0)
    ctx.set_nccl(_lib.nccl_unique_id(), 0, 1)
    st = _lib.tk_comm()
    st.rank, st.world = 0, 1
    st.blocked = 1
    for n, d in enumerate(dims):
        st.global_dims[n] = d
    _lib.check(lib.tk_context_set_comm(ctx.handle, C.byref(st)))
    runs = [P.rand_tucker_2i(yd, (8, 8, 8), 4, (1, 3), context=ctx, sync_ranks=False, out="host",
                             global_dims=dims) for _ in range(4)]  # eager, capture, 2 replays
    for m in runs:
        np.testing.assert_array_equal(m.core, ref.core)
        for u, v in zip(m.factors, ref.factors):
            np.testing.assert_array_equal(u, v)
    ctx.set_nccl(None)
    torch.cuda.synchronize()
