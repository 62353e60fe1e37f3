"""Streaming fit (tk_model_fit): fit(y, reconstruct(model)) (tensor.hpp:282-290,
tucker.hpp:63-66) and fit(y, cp_reconstruct(model)) (cp.hpp:118-128) against the oracle,
which materialises the reconstruction. fp64 data: 1e-12; fp32 data: the oracle on the same
fp32 values, 1e-9 (accumulation is fp64 on both sides)."""
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


@pytest.mark.parametrize("dims", [(40, 36, 30), (130, 70, 9), (12, 10, 8, 6), (70, 65)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_tucker_fit_matches_oracle(P, O, dims, dtype):
    ranks = tuple(min(4, d) for d in dims)
    seed = O.seed_derived(1, 2, 3)
    y = O.add_noise(O.gen_tucker(dims, ranks, seed), 12.0, O.seed_derived(*seed, 0xAD0)).astype(dtype)
    core = O.gaussian_matrix(int(np.prod(ranks)), 1, (4, 4)).reshape(ranks, order="F")
    fs = [O.gaussian_matrix(d, r, (5, n)) for n, (d, r) in enumerate(zip(dims, ranks))]
    ref = O.fit(y.astype(np.float64), O.reconstruct(core, fs))
    got = P.model_fit(P.DenseTensor.from_numpy(y, dtype), P.TuckerModel(core, fs, ranks))
    assert abs(got - ref) < (1e-12 if dtype == np.float64 else 1e-9)
    # the decomposition's own (device) model
    m = P.rand_tucker_2i(P.DenseTensor.from_numpy(y, dtype).cuda(), ranks, 2, (7, 0), out="device")
    h = m.to_host()
    ref2 = O.fit(y.astype(np.float64), O.reconstruct(h.core, h.factors))
    assert abs(P.model_fit(P.DenseTensor.from_numpy(y, dtype).cuda(), m) - ref2) < 1e-9


@pytest.mark.parametrize("dims", [(40, 36, 30), (12, 10, 8, 6)])
def test_cp_fit_matches_oracle(P, O, dims):
    fs = [np.abs(O.gaussian_matrix(d, 5, (8, n))) for n, d in enumerate(dims)]
    y = O.add_noise(O.cp_reconstruct(fs), 15.0, (9, 9))
    est = [f + 0.01 * O.gaussian_matrix(f.shape[0], 5, (10, n)) for n, f in enumerate(fs)]
    ref = O.fit(y, O.cp_reconstruct(est))
    got = P.model_fit(P.DenseTensor.from_numpy(y), P.CpModel(est))
    assert abs(got - ref) < 1e-12
    # FFCP output (device factors) feeds it directly
    g, us = O.rand_tucker_2i(y, (5,) * len(dims), 2, (11, 0))
    res = P.ffcp(P.TuckerModel(g, us, g.shape), 5, stop=P.StopRule(50, 1e-9), seed=(12, 0))
    assert abs(P.model_fit(P.DenseTensor.from_numpy(y), res) - O.fit(y, O.cp_reconstruct(res.factors))) < 1e-12


def test_fit_exact_model_is_one(P, O):
    dims, ranks = (50, 40, 30), (3, 3, 3)
    core = O.gaussian_matrix(27, 1, (1, 1)).reshape(ranks, order="F")
    fs = [O.gaussian_matrix(d, 3, (2, n)) for n, d in enumerate(dims)]
    y = O.reconstruct(core, fs)
    f, res, ny = P.model_fit(P.DenseTensor.from_numpy(y), P.TuckerModel(core, fs, ranks), norms=True)
    assert res <= 1e-13 * ny and abs(f - 1.0) < 1e-13


@pytest.mark.parametrize("c,R", [(40, 33), (60, 50), (64, 64)])
def test_ffcp_wide_ranks_match_oracle(P, O, c, R):
    """FFCP with R > 32 on large cores: (40^3, 33) runs the persistent kernel; (60^3, 50) and
    (64^3, 64) — whose shared-memory plan does not fit it — the captured sweep graph. Both
    follow ffcp.hpp:94-194 like the oracle (fit trace within 1e-8)."""
    rng = np.random.default_rng(c + R)
    g = rng.standard_normal((c, c, c))
    us = [np.linalg.qr(rng.standard_normal((c + 20, c)))[0] for _ in range(3)]
    _, tr_ref, it_ref = O.ffcp(g, us, R, O.NONE, 0.0, 12, 0.0, (5, 0))
    res = P.ffcp(P.TuckerModel(g, us, g.shape), R, stop=P.StopRule(12, 0.0), seed=(5, 0))
    assert res.iterations == it_ref
    np.testing.assert_allclose(res.fit_trace, tr_ref, rtol=0, atol=1e-8)
