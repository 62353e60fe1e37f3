"""The second-design Y-streaming kernel (csrc/ttm_stream.cu: [y_hi | y_lo] A operands from TMEM,
chunked accumulation flushed into fp32 registers)
against the oracle's ttm (tensor.hpp:151-176) and the FFMA kernel, through tk_ttm with
ttm path 3 (M-major contractions), and inside rand_tucker_2i, where it runs every Y pass
(M-major and the mode-0 K-major pass with its transposed output).

Bar: fp32 accumulation level, as for the first tcgen05 kernel (3e-6 sqrt(K/100 + 1) relative);
the chunked accumulation keeps the error flat in K (checked at K = 4000)."""
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


@pytest.mark.parametrize("shape,mode", [((512, 300, 300), 1), ((1024, 100, 80), 1), ((2048, 333, 40), 1),
                                        ((300, 400, 64), 2), ((256, 4000, 300), 1),
                                        # tiles of 128 p x 2 q (ragged P: fewer idle tile rows), odd / even Q
                                        ((640, 64, 301), 1), ((2400, 48, 40), 1)])
@pytest.mark.parametrize("rows", [8, 15, 20, 30, 40, 50, 60, 64])
def test_stream_ttm_matches_oracle_and_ffma(P, O, shape, mode, rows):
    ctx = P.Context.default()
    t = O.gaussian_matrix(int(np.prod(shape)), 1, (5, rows)).reshape(shape, order="F").astype(np.float32)
    m = O.gaussian_matrix(rows, shape[mode], (6, rows))
    ref = O.ttm(t.astype(np.float64), m, mode)
    try:
        ctx.set_ttm_path("stream")
        got = P.ttm(P.DenseTensor.from_numpy(t, np.float32), m, mode)
        ctx.set_ttm_path("ffma")
        got_ffma = P.ttm(P.DenseTensor.from_numpy(t, np.float32), m, mode)
    finally:
        ctx.set_ttm_path("auto")
    k = shape[mode]
    tol = 3e-6 * np.sqrt(k / 100 + 1)
    assert rel(got, ref) < tol, (rel(got, ref), tol)
    assert rel(got_ffma, ref) < tol
    # the chunked accumulation: no growth of the error with K (K = 4000: at the FFMA kernel's level)
    if k >= 4000:
        assert rel(got, ref) < 2 * rel(got_ffma, ref) + 1e-7


@pytest.mark.parametrize("ranks,p", [((50, 50, 50), 10), ((15, 15, 15), 5)])
def test_rand_tucker_2i_stream_passes_match_oracle(P, O, ranks, p):
    """400^3 fp32: every Y pass on the streaming kernel (M-major passes and the mode-0 K-major
    pass writing its output transposed); r~ = 60 (NH 64, one tile per CTA) and r~ = 20 (NH 24)."""
    seed = (8, 1)
    dims = (400, 400, 400)
    y = O.add_noise(O.gen_tucker(dims, (10, 10, 10), seed), 20.0, O.seed_derived(*seed, 0xAD0))
    y32 = y.astype(np.float32)
    import os
    O.set_threads(os.cpu_count() or 1)
    g_ref, u_ref = O.rand_tucker_2i(y32.astype(np.float64), ranks, p, (7, 2))
    O.set_threads(1)
    m = P.rand_tucker_2i(P.DenseTensor.from_numpy(y32, np.float32).cuda(), ranks, p, (7, 2), sync_ranks=False).to_host()
    assert m.stats["passes"] == 3
    for u, v in zip(m.factors, u_ref):
        assert u.shape == v.shape
        assert orthonormality_defect(u) < 1e-10
        assert subspace_dist(u, v) < 1e-3
    aligned = O.ttm_all(m.core, [u.T @ v for u, v in zip(m.factors, u_ref)], -1, False)
    assert rel(aligned, g_ref) < 1e-3


@pytest.mark.parametrize("dims,ranks,p", [((60, 50, 40), (5, 5, 5), 4), ((704, 700, 640), (12, 12, 12), 8)])
def test_fp64_mode_on_fp32_data_matches_oracle_at_fp64_bar(P, O, dims, ranks, p):
    """precision='fp64': fp64 arithmetic over fp32 values — a cast copy for small tensors, the
    mixed fp32-in / fp64 kernel (ttm_mixed.cu) for tensors whose fp64 copy exceeds 2 GB (the
    second case) — equals the oracle on the same values at the fp64 bar, factor by factor."""
    import os
    import torch
    from paper_1412_1885_b200.generators import generate_as
    cfg = dict(dims=dims, gen="tucker", mlrank=(6, 6, 6), snr=20.0, seed=3)
    y32 = generate_as(cfg, torch.float32)
    m = P.rand_tucker_2i(P.DenseTensor(dims, y32), ranks, p, (2, 9), sync_ranks=False, out="host", precision="fp64")
    m2 = P.rand_tucker_2i(P.DenseTensor(dims, y32), ranks, p, (2, 9), sync_ranks=False, out="host", precision="fp64")
    yh = y32.cpu().numpy()
    O.set_threads(os.cpu_count() or 1)
    g_ref, u_ref, _ = O.rand_tucker_2i_streamed(yh, dims, ranks, p, (2, 9))
    O.set_threads(1)
    for u, v, w in zip(m.factors, u_ref, m2.factors):
        np.testing.assert_array_equal(u, w)  # deterministic (second call: graph replay)
        assert u.shape == v.shape and np.abs(u - v).max() < 1e-8
    assert rel(m.core, g_ref) < 1e-8
    assert m.stats["y_bytes"] == 4 * int(np.prod(dims))


def test_host_input_lands_in_slabs_under_the_first_pass(P, O):
    """Host input (the e2e path, bench.hpp:456-520 times the copy-in): the tensor is copied in
    last-mode slabs on a copy stream and the first Y pass (leader = last mode) multiplies each
    slab as it lands, partial sums added in slab order. Same model as the device-input call up to
    fp32 rounding of the slab sums, and the oracle's within the fp32 bar."""
    import torch
    seed = (8, 3)
    dims = (416, 400, 208)
    ranks, p = (12, 12, 12), 8
    y = O.add_noise(O.gen_tucker(dims, (10, 10, 10), seed), 20.0, O.seed_derived(*seed, 0xAD0))
    y32 = y.astype(np.float32)
    import os
    O.set_threads(os.cpu_count() or 1)
    g_ref, u_ref = O.rand_tucker_2i(y32.astype(np.float64), ranks, p, (7, 4))
    O.set_threads(1)
    host = P.DenseTensor.from_numpy(y32, np.float32)
    m_host = P.rand_tucker_2i(host, ranks, p, (7, 4), sync_ranks=False, out="host")
    m_dev = P.rand_tucker_2i(host.cuda(), ranks, p, (7, 4), sync_ranks=False).to_host()
    assert m_host.stats["passes"] == 3 and m_dev.stats["passes"] == 3
    # 208 / 8 slabs -> 32-k ranges: 7 launches of the first pass instead of 1
    assert m_host.stats["kernel_launches"] == m_dev.stats["kernel_launches"] + 6
    for uh, ud, v in zip(m_host.factors, m_dev.factors, u_ref):
        assert uh.shape == ud.shape == v.shape
        assert subspace_dist(uh, ud) < 2e-4
        assert subspace_dist(uh, v) < 1e-3
        assert orthonormality_defect(uh) < 1e-10
    aligned = O.ttm_all(m_host.core, [u.T @ v for u, v in zip(m_host.factors, u_ref)], -1, False)
    assert rel(aligned, g_ref) < 1e-3
    # twice in a row (the landing buffer is reused while the copy stream refills it)
    m2 = P.rand_tucker_2i(host, ranks, p, (7, 4), sync_ranks=False, out="host")
    for a, b in zip(m_host.factors, m2.factors):
        assert np.array_equal(a, b)
    assert np.array_equal(m_host.core, m2.core)
