"""Parity of the sm_100a path against the CPU oracle (oracle/), through the C-ABI.

Bars (north star): subspaces ||U U^T - U' U'^T||_F, the aligned core and the fit agree
within 1e-5 in fp64 (Y fp64) and 1e-3 in fp32 (Y fp32, oracle in fp64 on the same fp32
values). Kernel-level results are compared at fp64 rounding level (<= 1e-12 relative) or
fp32 accumulation level (<= 2e-5 relative)."""
import numpy as np
import pytest

from helpers import orthonormality_defect, subspace_dist, transpositions_to_perm

pytestmark = pytest.mark.gpu

F64_TOL = 1e-5
F32_TOL = 1e-3


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1412_1885_b200 as P
    return P


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def rt(O, shape, seed):
    return O.gaussian_matrix(int(np.prod(shape)), 1, (seed, 0)).reshape(shape, order="F")


def noisy_tucker(O, dims, ranks, snr_db, seed):
    y = O.gen_tucker(dims, ranks, seed)
    return O.add_noise(y, snr_db, O.seed_derived(*seed, 0xAD0))


# ------------------------------------------------------------------ RNG / kernels
def test_gaussian_matrix_matches_oracle(P, O):
    for rows, cols, seed in [(7, 4, (5, 11)), (1000, 30, (0, 3)), (999, 3, (1, 2))]:
        d = P.gaussian_matrix(rows, cols, seed)
        h = O.gaussian_matrix(rows, cols, seed)
        assert np.max(np.abs(d - h)) <= 4e-15 * max(1.0, np.max(np.abs(h)))


@pytest.mark.parametrize("shape", [(200, 40, 30), (64, 33, 17), (3, 4, 2), (12, 10, 9, 8), (256, 300), (5, 4000)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_ttm_all_modes(P, O, shape, dtype):
    import torch
    t = rt(O, shape, 8)
    tt = P.DenseTensor.from_numpy(t, np.float32 if dtype == "f32" else np.float64)
    for n in range(len(shape)):
        for rows in (1, 5, 15, 30, 64):
            m = O.gaussian_matrix(rows, shape[n], (9, n + rows))
            ref = O.ttm(tt.numpy().astype(np.float64), m, n)
            got = P.ttm(tt, m, n)
            assert rel(got, ref) < (1e-12 if dtype == "f64" else 2e-5 * np.sqrt(shape[n] / 100 + 1))


@pytest.mark.parametrize("shape,skip", [((60, 50, 40), -1), ((60, 50, 40), 0), ((60, 50, 40), 1), ((60, 50, 40), 2),
                                        ((20, 18, 16, 14), 3), ((20, 18, 16, 14), 1)])
def test_ttm_all_projection(P, O, shape, skip):
    t = rt(O, shape, 13)
    us = [O.gaussian_matrix(s, 7, (14, k)) for k, s in enumerate(shape)]
    ref = O.ttm_all(t, us, skip, True)
    got = P.ttm_all(P.DenseTensor.from_numpy(t), us, skip)
    assert rel(got, ref) < 1e-12


@pytest.mark.parametrize("skip", [2, -1])
def test_ttm_all_mode0_first_stage_fp32(P, O, skip):
    """fp32 shapes whose first (Y-streaming) contraction is over mode 0 (I_0 < 256: no
    M-major pass over mode 1): the K-major tcgen05 pass writes its output transposed (mode 0
    last) and ttm_all returns the standard layout."""
    shape = (200, 300, 160)
    t = rt(O, shape, 17).astype(np.float32)
    us = [O.gaussian_matrix(s, 12, (15, k)) for k, s in enumerate(shape)]
    ref = O.ttm_all(t.astype(np.float64), us, skip, True)
    got = P.ttm_all(P.DenseTensor.from_numpy(t, np.float32), us, skip)
    assert got.shape == ref.shape
    assert rel(got, ref) < 1e-5


@pytest.mark.parametrize("shape", [(40, 30, 20), (7, 9, 11), (10, 9, 8, 7)])
def test_unfold_times(P, O, shape):
    t = rt(O, shape, 11)
    for n in range(len(shape)):
        b = O.gaussian_matrix(t.size // t.shape[n], 6, (12, n))
        assert rel(P.unfold_times(P.DenseTensor.from_numpy(t), n, b), O.unfold_times(t, n, b)) < 1e-12


# ------------------------------------------------------------------ pivoted QR
@pytest.mark.parametrize("rows,cols", [(50, 8), (200, 15), (1000, 30), (2400, 40), (300, 20), (31, 31), (4000, 60),
                                       (12, 1)])
def test_orthonormal_basis_matches_oracle(P, O, rows, cols):
    z = O.gaussian_matrix(rows, cols, (rows, cols))
    if cols > 2:
        z[:, 1] = 3.0 * z[:, 0] + 1e-3 * z[:, 1]  # exercises the norm downdate / recompute path
    u_ref, d = O.orthonormal_basis(z, diagnostics=True)
    u_ref = O.fix_column_signs(u_ref)
    u, diag = P.orthonormal_basis(z, with_diag=True)
    assert u.shape == u_ref.shape
    assert np.allclose(np.abs(diag), np.abs(d["rdiag"]), rtol=1e-10, atol=1e-12)  # same pivots, same R_kk
    assert np.max(np.abs(u - u_ref)) < 1e-10
    assert orthonormality_defect(u) < 1e-12


def test_orthonormal_basis_rank_deficient_and_zero(P, O):
    z = np.zeros((5, 2))
    z[0, 0], z[0, 1] = 1.0, 2.0
    u = P.orthonormal_basis(z)
    assert u.shape == (5, 1) and abs(abs(u[0, 0]) - 1.0) < 1e-14
    assert P.orthonormal_basis(np.zeros((6, 3))).shape == (6, 0)
    m = O.gaussian_matrix(40, 6, (3, 0)) @ O.gaussian_matrix(6, 16, (3, 1))
    u = P.orthonormal_basis(m)
    u_ref = O.fix_column_signs(O.orthonormal_basis(m))
    assert u.shape == u_ref.shape == (40, 6)
    assert subspace_dist(u, u_ref) < 1e-10


# ------------------------------------------------------------------ Tucker drivers
def compare_models(O, y, got, ref, tol):
    g_ref, us_ref = ref
    assert [u.shape[1] for u in got.factors] == [u.shape[1] for u in us_ref]
    for u, v in zip(got.factors, us_ref):
        assert subspace_dist(u, v) < tol * max(1.0, np.sqrt(v.shape[1]))
        assert orthonormality_defect(u) < 1e-10
    # core after aligning bases: G x_n (U_n^T U'_n)
    aligned = O.ttm_all(got.core, [u.T @ v for u, v in zip(got.factors, us_ref)], -1, False)
    assert rel(aligned, g_ref) < tol
    f_got = O.fit(y, O.reconstruct(got.core, got.factors))
    f_ref = O.fit(y, O.reconstruct(g_ref, us_ref))
    assert abs(f_got - f_ref) < tol


@pytest.mark.parametrize("dims,ranks,p,snr", [((40, 36, 30), (5, 4, 3), 5, 10.0), ((24, 24, 24, 24), (3, 3, 3, 3), 4, 20.0),
                                              ((64, 50), (6, 5), 4, 10.0), ((300, 12, 10), (4, 4, 4), 3, 5.0)])
def test_rand_tucker_2i_f64_matches_oracle(P, O, dims, ranks, p, snr):
    y = noisy_tucker(O, dims, ranks, snr, (1, 2))
    seed = (33, 0)
    ref = O.rand_tucker_2i(y, ranks, p, seed)
    got = P.rand_tucker_2i(y, ranks, p, seed)
    compare_models(O, y, got, ref, F64_TOL)
    # bitwise determinism (reference test_tucker.cpp:108-117)
    again = P.rand_tucker_2i(y, ranks, p, seed)
    assert np.array_equal(again.core, got.core)


def test_config1_cpu_runnable_case(P, O):
    """BASELINE config 1: 200^3 fp64 rank-10 CP with U(0,1) factors + noise at 10 dB,
    ranks (10,10,10), oversample 5; then FFCP rank 10 (bench.hpp seeds, cfg.seed=0)."""
    root = (0, 0)
    data = O.seed_derived(*root, 0xDA7A, 0)
    alg = O.seed_derived(*root, 0xA16D, 0)
    y, _ = O.gen_cp((200, 200, 200), 10, O.CP_UNIFORM, data)
    y = O.add_noise(y, 10.0, O.seed_derived(*data, 0xAD0))
    ref = O.rand_tucker_2i(y, (10, 10, 10), 5, alg)
    got = P.rand_tucker_2i(y, (10, 10, 10), 5, alg)
    compare_models(O, y, got, ref, F64_TOL)
    a_ref, tr_ref, it_ref = O.ffcp(ref[0], ref[1], 10, O.NONE, 0.0, 200, 1e-6, alg)
    res = P.ffcp(got, 10, stop=P.StopRule(200, 1e-6), seed=alg)
    assert abs(res.fit_trace[-1] - tr_ref[-1]) < F64_TOL
    f_ref = O.fit(y, O.cp_reconstruct(a_ref))
    f_got = O.fit(y, O.cp_reconstruct(res.factors))
    assert abs(f_got - f_ref) < F64_TOL


@pytest.mark.parametrize("dims,ranks,p", [((128, 96, 80), (8, 8, 8), 6), ((60, 52, 48, 40), (4, 4, 4, 4), 4)])
def test_rand_tucker_2i_f32_matches_oracle(P, O, dims, ranks, p):
    y = noisy_tucker(O, dims, ranks, 20.0, (3, 4)).astype(np.float32).astype(np.float64)
    seed = (34, 0)
    ref = O.rand_tucker_2i(y, ranks, p, seed)
    got = P.rand_tucker_2i(y.astype(np.float32), ranks, p, seed)
    compare_models(O, y, got, ref, F32_TOL)


def test_rand_tucker_2i_exact_rank_drop(P, O):
    """Noise-free multilinear rank 5 with r~ = 15: the rank cut drops 10 columns (test_tucker.cpp:108-117)."""
    core = rt(O, (5, 5, 5), 1)
    us = [O.gaussian_matrix(30, 5, (32, 2 + n)) for n in range(3)]
    y = O.reconstruct(core, us)
    ref = O.rand_tucker_2i(y, (5, 5, 5), 10, (33, 0))
    for sync in (True, False):
        got = P.rand_tucker_2i(y, (5, 5, 5), 10, (33, 0), sync_ranks=sync)
        assert [u.shape[1] for u in got.factors] == [5, 5, 5]
        assert O.fit(y, O.reconstruct(got.core, got.factors)) > 1 - 1e-8
        compare_models(O, y, got, ref, F64_TOL)


def test_speculative_and_explicit_core_agree(P, O):
    y = noisy_tucker(O, (50, 40, 30), (5, 5, 5), 10.0, (5, 6))
    a = P.rand_tucker_2i(y, (5, 5, 5), 5, (7, 0))
    b = P.rand_tucker_2i(y, (5, 5, 5), 5, (7, 0), sync_ranks=False)
    c = P.rand_tucker_2i(y, (5, 5, 5), 5, (7, 0), explicit_core_pass=True)
    assert np.array_equal(a.core, b.core)
    assert rel(c.core, a.core) < 1e-12
    # consecutive steps share a Y pass: 3 passes (+1 for the explicit core) instead of 6 (7)
    assert a.stats["passes"] == 3 and c.stats["passes"] == 4


@pytest.mark.parametrize("dims,dtype", [((50, 40, 30), np.float64), ((300, 280, 260), np.float32),
                                        ((24, 22, 20, 18), np.float64), ((40, 36, 30, 28), np.float32)])
def test_shared_passes_match_one_pass_per_step(P, O, dims, dtype):
    """Grouped steps (one Y pass shared by consecutive range steps, N = 3: 3 passes, N = 4: 3)
    == the reference's one-pass-per-step structure (tucker.hpp:149-160) == the oracle."""
    order = len(dims)
    ranks = (4,) * order
    y = noisy_tucker(O, dims, ranks, 15.0, (21, order))
    yy = P.DenseTensor.from_numpy(y.astype(dtype), dtype).cuda() if dtype == np.float32 else y
    g = P.rand_tucker_2i(yy, ranks, 3, (8, 1), out="host")
    s = P.rand_tucker_2i(yy, ranks, 3, (8, 1), out="host", one_pass_per_step=True)
    assert g.stats["passes"] == 3 and s.stats["passes"] == 2 * order
    ref = O.rand_tucker_2i(y.astype(dtype).astype(np.float64), ranks, 3, (8, 1))
    # fp32: the two contraction orders round differently; both sit ~1e-4 from the fp64 oracle
    # in the noise directions, so they are held to the north star's fp32 bar (1e-3)
    tol = 1e-10 if dtype == np.float64 else F32_TOL
    for u, v in zip(g.factors, s.factors):
        assert subspace_dist(u, v) < tol
    compare_models(O, y, g, ref, F64_TOL if dtype == np.float64 else F32_TOL)


def test_device_resident_path(P, O):
    import torch
    y = noisy_tucker(O, (80, 70, 60), (6, 6, 6), 20.0, (8, 9))
    yd = P.DenseTensor.from_numpy(y, np.float32).cuda()
    m = P.rand_tucker_2i(yd, (6, 6, 6), 4, (10, 0))
    assert m.core.is_cuda
    h = m.to_host()
    ref = O.rand_tucker_2i(y.astype(np.float32).astype(np.float64), (6, 6, 6), 4, (10, 0))
    compare_models(O, y, h, ref, F32_TOL)


def test_rand_tucker_alg2_matches_oracle(P, O):
    y = noisy_tucker(O, (60, 50, 40), (5, 5, 5), 10.0, (11, 12))
    ref = O.rand_tucker(y, (5, 5, 5), 5, (13, 0))
    got = P.rand_tucker(y, (5, 5, 5), 5, (13, 0))
    compare_models(O, y, got, ref, F64_TOL)


@pytest.mark.parametrize("dims,mlr,ranks,p", [((400, 400, 400), (10, 10, 10), (20, 20, 20), 10),
                                              ((640, 300, 280), (8, 8, 8), (30, 12, 12), 10),
                                              ((72, 64, 60, 56), (4, 4, 4, 4), (6, 6, 6, 6), 4)])
def test_rand_tucker_alg2_fp32_workload_shapes_match_oracle(P, O, dims, mlr, ranks, p):
    """Alg. 2 (tucker.hpp:108-130) in fp32 at shapes whose first (Y-streaming) contraction runs
    on the tensor-core kernels, 3- and 4-way, against the fp64 oracle on the fp32 values."""
    import os
    y = noisy_tucker(O, dims, mlr, 20.0, (31, len(dims))).astype(np.float32)
    O.set_threads(os.cpu_count() or 1)
    ref = O.rand_tucker(y.astype(np.float64), ranks, p, (32, 0))
    O.set_threads(1)
    got = P.rand_tucker(P.DenseTensor.from_numpy(y, np.float32).cuda(), ranks, p, (32, 0)).to_host()
    compare_models(O, y.astype(np.float64), got, ref, F32_TOL)


def test_ffcp_variants_match_oracle(P, O):
    fs = [np.abs(O.gaussian_matrix(d, 3, (84, n))) for n, d in enumerate((10, 9, 8))]
    y = O.cp_reconstruct(fs)
    g, us = O.rand_tucker_2i(y, (3, 3, 3), 5, (85, 0))
    model = P.TuckerModel(g, us, g.shape)
    for kind in (O.NONE, O.NONNEG_MU, O.NONNEG_HALS, O.SPARSE):
        a_ref, tr_ref, it_ref = O.ffcp(g, us, 3, kind, 0.05, 30, 0.0, (86, 0))
        res = P.ffcp(model, 3, P.ConstraintSpec(kind, 0.05), P.StopRule(30, 0.0), (86, 0))
        assert res.iterations == it_ref
        assert np.allclose(res.fit_trace, tr_ref, rtol=1e-9, atol=1e-9)
        for a, b in zip(res.factors, a_ref):
            assert np.allclose(a, b, rtol=1e-7, atol=1e-9)


def test_ffcp_device_model_matches_oracle(P, O):
    """FFCP straight on the device outputs of rand_tucker_2i (no host round trip), 4-way
    nonnegative HALS (BASELINE config 4's constraint) and unconstrained."""
    fs = [np.abs(O.gaussian_matrix(d, 3, (90, n))) for n, d in enumerate((14, 12, 10, 9))]
    y = O.add_noise(O.cp_reconstruct(fs), 30.0, (91, 0), abs_noise=True)
    m = P.rand_tucker_2i(P.DenseTensor.from_numpy(y).cuda(), (3, 3, 3, 3), 2, (92, 0))
    h = m.to_host()
    for kind in (O.NONNEG_HALS, O.NONE):
        res = P.ffcp(m, 3, P.ConstraintSpec(kind), P.StopRule(200, 1e-6), (93, 0))
        a_ref, tr_ref, it_ref = O.ffcp(h.core, h.factors, 3, kind, 0.0, 200, 1e-6, (93, 0))
        assert res.iterations == it_ref
        assert np.allclose(res.fit_trace, tr_ref, rtol=1e-8, atol=1e-8)
        assert abs(O.fit(y, O.cp_reconstruct(res.factors)) - O.fit(y, O.cp_reconstruct(a_ref))) < 1e-6


def test_errors_mirror_reference(P):
    with pytest.raises(P.TenkitError, match="one rank per mode required"):
        P.rand_tucker_2i(np.ones((3, 3, 3)), (2, 2), 1, (0, 0))
    with pytest.raises(P.TenkitError, match="tensor dimensions must be positive"):
        P.rand_tucker_2i(np.zeros((6, 5, 4)), (2, 2, 2), 1, (0, 0))  # zero data: rank-0 factor


def test_repeated_calls_replay_graph_identically(P, O):
    """A repeated rand_tucker_2i call is captured as a CUDA graph and replayed: every
    replay returns the bit-identical model of the eager call, kernel timing still works, and
    a call that reallocates the context's buffers in between invalidates the graph."""
    import torch
    dims = (300, 280, 260)
    y = O.add_noise(O.gen_tucker(dims, (6, 6, 6), (3, 3)), 20.0, (4, 4)).astype(np.float32)
    yd = P.DenseTensor.from_numpy(y, np.float32).cuda()
    ctx = P.Context.default()
    runs = [P.rand_tucker_2i(yd, (6, 6, 6), 4, (9, 0), sync_ranks=False, out="device", time_kernels=True).to_host()
            for _ in range(4)]
    for m in runs[1:]:
        np.testing.assert_array_equal(m.core, runs[0].core)
        for a, b in zip(m.factors, runs[0].factors):
            np.testing.assert_array_equal(a, b)
        assert m.stats["stream_ms"] > 0 and m.stats["passes"] == 3
    big = P.DenseTensor.from_numpy(np.ones((400, 390, 380), np.float32), np.float32).cuda()
    P.rand_tucker_2i(big, (6, 6, 6), 4, (9, 0), sync_ranks=False, out="device")  # grows the buffers
    again = P.rand_tucker_2i(yd, (6, 6, 6), 4, (9, 0), sync_ranks=False, out="device").to_host()
    np.testing.assert_array_equal(again.core, runs[0].core)
    del big
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dims,ranks,p,dtype", [
    ((5, 40, 30), (10, 4, 4), 2, np.float64),       # R + p >= I_0: r~_0 clamped to I_0 (square factor)
    ((50,), (3,), 2, np.float64),                    # order 1
    ((6, 5, 4, 5, 6), (2, 2, 2, 2, 2), 1, np.float64),  # order 5
    ((40, 36, 30), (5, 4, 3), 0, np.float64),        # no oversampling
    ((37, 41, 43), (4, 5, 3), 3, np.float32),        # fp32, extents not multiples of 4 (FFMA paths)
    ((200, 100, 70), (60, 10, 10), 4, np.float64),   # r~ = 64, the device maximum
])
def test_edge_shapes_match_oracle(P, O, dims, ranks, p, dtype):
    y = noisy_tucker(O, dims, tuple(min(r, d) for r, d in zip(ranks, dims)), 15.0, (5, 6)).astype(dtype)
    seed = (21, 0)
    ref = O.rand_tucker_2i(y.astype(np.float64), ranks, p, seed)
    got = P.rand_tucker_2i(P.DenseTensor.from_numpy(y, dtype), ranks, p, seed)
    compare_models(O, y.astype(np.float64), got, ref, F64_TOL if dtype == np.float64 else F32_TOL)
    ref2 = O.rand_tucker(y.astype(np.float64), ranks, p, seed)
    got2 = P.rand_tucker(P.DenseTensor.from_numpy(y, dtype), ranks, p, seed)
    compare_models(O, y.astype(np.float64), got2, ref2, F64_TOL if dtype == np.float64 else F32_TOL)


def test_device_rank_limit_is_an_error(P, O):
    y = rt(O, (200, 100, 70), 3)
    with pytest.raises(P.TenkitError, match="rank \\+ oversample must be <= 64"):
        P.rand_tucker_2i(y, (61, 10, 10), 4, (1, 0))
