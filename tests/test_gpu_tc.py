"""The tcgen05 (UMMA, 3xTF32) Y-streaming TTM kernel against the oracle and the FFMA kernel.

3xTF32 keeps ~2^-21 relative error per product (plain TF32 is not
fp32-accurate enough for basis parity); the bar is fp32 accumulation level."""
import numpy as np
import pytest

from helpers import orthonormality_defect, subspace_dist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1412_1885_b200 as P
    return P


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


@pytest.mark.parametrize("shape,mode", [((512, 40, 300), 1), ((1000, 37, 320), 1), ((256, 1000, 300), 1),
                                        ((600, 500, 8), 2),
                                        # mode 0 (K-major tcgen05 variant): 128-row and 512-row tiles
                                        ((64, 300, 80), 0), ((1000, 40, 600), 0), ((100, 613, 37), 0),
                                        ((20, 400, 400), 0)])
@pytest.mark.parametrize("rows", [8, 15, 30, 40, 64])
def test_tc_ttm_matches_oracle_and_ffma(P, O, shape, mode, rows):
    import torch
    ctx = P.Context.default()
    t = O.gaussian_matrix(int(np.prod(shape)), 1, (3, rows)).reshape(shape, order="F").astype(np.float32)
    m = O.gaussian_matrix(rows, shape[mode], (4, rows))
    ref = O.ttm(t.astype(np.float64), m, mode)
    try:
        ctx.set_ttm_path("tc")
        got_tc = P.ttm(P.DenseTensor.from_numpy(t, np.float32), m, mode)
        ctx.set_ttm_path("ffma")
        got_ffma = P.ttm(P.DenseTensor.from_numpy(t, np.float32), m, mode)
    finally:
        ctx.set_ttm_path("auto")
    k = shape[mode]
    tol = 3e-6 * np.sqrt(k / 100 + 1)
    assert rel(got_tc, ref) < tol
    assert rel(got_ffma, ref) < tol
    assert rel(got_tc, got_ffma) < 2 * tol


@pytest.mark.parametrize("ranks,p", [((12, 12, 12), 8), ((30, 30, 30), 10)])
def test_rand_tucker_2i_tc_path_matches_oracle(P, O, ranks, p):
    """400^3 fp32 (first-stage tiles >= 2 waves -> tcgen05 path in auto mode); r~ = 20 and 40
    (the mode-0 Y pass on the K-major kernel with NH = 32 and NH = 48)."""
    seed = (5, 6)
    dims = (400, 400, 400)
    y = O.add_noise(O.gen_tucker(dims, ranks, seed), 20.0, O.seed_derived(*seed, 0xAD0))
    y32 = y.astype(np.float32)
    O.set_threads(8)
    g_ref, u_ref = O.rand_tucker_2i(y32.astype(np.float64), ranks, p, (7, 0))
    O.set_threads(1)
    ctx = P.Context.default()
    ctx.set_ttm_path("auto")
    m = P.rand_tucker_2i(P.DenseTensor.from_numpy(y32, np.float32).cuda(), ranks, p, (7, 0), sync_ranks=False).to_host()
    for u, v in zip(m.factors, u_ref):
        assert orthonormality_defect(u) < 1e-10
        assert subspace_dist(u, v) < 1e-3
    ysq = float(np.sum(y32.astype(np.float64) ** 2))
    assert abs(float(np.sum(m.core ** 2)) - float(np.sum(g_ref ** 2))) / ysq < 1e-5
    assert m.stats["passes"] == 3  # steps share Y passes; the mode-0 pass on the K-major kernel


@pytest.mark.parametrize("dims", [(64, 150, 150), (128, 160, 120)])
def test_rand_tucker_2i_wide_kmajor_leader_matches_oracle(P, O, dims):
    """r~ = 60 (ranks 50, p 10): mode 0 leads a Y pass on the NH = 64 K-major tcgen05 kernel
    (one CTA per SM, 3 accumulator sets) with the transposed output (tout), fp32 vs the oracle."""
    seed = (3, 9)
    ranks, p = (50, 50, 50), 10
    y = O.add_noise(O.gen_tucker(dims, (12, 12, 12), seed), 20.0, O.seed_derived(*seed, 0xAD0))
    y32 = y.astype(np.float32)
    O.set_threads(8)
    g_ref, u_ref = O.rand_tucker_2i(y32.astype(np.float64), ranks, p, (7, 1))
    O.set_threads(1)
    m = P.rand_tucker_2i(P.DenseTensor.from_numpy(y32, np.float32).cuda(), ranks, p, (7, 1), sync_ranks=False).to_host()
    assert m.stats["passes"] == 3
    for u, v in zip(m.factors, u_ref):
        assert u.shape == v.shape == (u.shape[0], min(60, u.shape[0]))
        assert orthonormality_defect(u) < 1e-10
        assert subspace_dist(u, v) < 1e-3
    aligned = O.ttm_all(m.core, [u.T @ v for u, v in zip(m.factors, u_ref)], -1, False)
    assert rel(aligned, g_ref) < 1e-3
