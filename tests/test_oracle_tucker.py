"""Pins the oracle's range finder, Tucker drivers and FFCP against the reference suite.

Mirrors /root/reference/proj/tests/test_range_finder.cpp, test_tucker.cpp, test_ffcp.cpp,
and pins the Eigen-ColPivHouseholderQR restatement against LAPACK dgeqp3 (scipy), the
published algorithm Eigen restates (pivot order + R diagonal + Q up to column sign)."""
import numpy as np
import pytest
import scipy.linalg as sl

from helpers import (max_principal_angle, orthonormality_defect, subspace_dist,
                     transpositions_to_perm)


def low_mlrank(O, dims, ranks, seed):  # test_support.hpp:45-54
    core = O.gaussian_matrix(int(np.prod(ranks)), 1, (seed, 1)).reshape(ranks, order="F")
    us = [O.gaussian_matrix(d, r, (seed, 2 + n)) for n, (d, r) in enumerate(zip(dims, ranks))]
    return O.reconstruct(core, us)


def rt(O, shape, seed):
    return O.gaussian_matrix(int(np.prod(shape)), 1, (seed, 0)).reshape(shape, order="F")


# ------------------------------------------------------------------ range_finder.hpp
def test_orthonormal_input_keeps_range(O):  # test_range_finder.cpp:10-17
    z = np.linalg.qr(O.gaussian_matrix(12, 4, (1, 0)))[0]
    q = O.orthonormal_basis(z)
    assert q.shape[1] == 4
    assert np.abs(q.T @ q - np.eye(4)).max() < 1e-12
    assert np.linalg.norm(z @ z.T - q @ q.T) < 1e-10


def test_drops_deficient_columns(O):  # test_range_finder.cpp:19-29
    z = np.zeros((5, 2))
    z[0, 0], z[0, 1] = 1.0, 2.0
    q = O.orthonormal_basis(z)
    assert q.shape[1] == 1 and abs(abs(q[0, 0]) - 1.0) < 1e-14
    assert O.orthonormal_basis(np.zeros((6, 3))).shape[1] == 0


def test_projection_residual(O):  # test_range_finder.cpp:31-35
    z = O.gaussian_matrix(50, 5, (2, 0))
    q = O.orthonormal_basis(z)
    assert np.linalg.norm(z - q @ (q.T @ z)) < 1e-10


def test_range_finder_exact_rank(O):  # test_range_finder.cpp:37-43
    m = O.gaussian_matrix(40, 6, (3, 0)) @ O.gaussian_matrix(6, 60, (3, 1))
    q = O.orthonormal_basis(m @ O.gaussian_matrix(60, 16, (3, 2)))
    assert np.linalg.norm(m - q @ (q.T @ m)) / np.linalg.norm(m) < 1e-10


def test_range_finder_zero(O):  # test_range_finder.cpp:45-48
    assert O.orthonormal_basis(np.zeros((10, 8)) @ O.gaussian_matrix(8, 3, (4, 0))).shape[1] == 0


def test_range_finder_within_2x_svd(O):  # test_range_finder.cpp:50-64
    m = O.gaussian_matrix(30, 4, (5, 0)) @ O.gaussian_matrix(4, 25, (5, 1)) + 0.01 * O.gaussian_matrix(30, 25, (5, 2))
    u = np.linalg.svd(m)[0][:, :4]
    svd_res = np.linalg.norm(m - u @ (u.T @ m))
    q = O.orthonormal_basis(m @ O.gaussian_matrix(25, 14, (5, 3)))
    assert np.linalg.norm(m - q @ (q.T @ m)) < 2 * svd_res + 1e-12


@pytest.mark.parametrize("rows,cols,seed", [(50, 8, 2), (200, 15, 3), (1000, 30, 4), (31, 31, 5), (300, 20, 6)])
def test_colpiv_matches_lapack_dgeqp3(O, rows, cols, seed):
    """Pin: pivot order, |R_kk| and Q (up to column sign) equal LAPACK's pivoted QR."""
    z = O.gaussian_matrix(rows, cols, (seed, 9))
    z[:, 1] = z[:, 0] * 3.0 + 1e-3 * z[:, 1]  # an ill-conditioned pair exercises norm downdating
    u, d = O.orthonormal_basis(z, diagnostics=True)
    q, r, p = sl.qr(z, mode="economic", pivoting=True)
    assert transpositions_to_perm(d["perm"]) == list(p)
    assert np.allclose(np.abs(d["rdiag"]), np.abs(np.diag(r)), rtol=1e-10, atol=1e-12)
    assert np.abs(np.abs(u) - np.abs(q[:, : u.shape[1]])).max() < 1e-10


def test_sign_rule(O):  # tucker.hpp:39-45
    u = np.array([[0.1, -3.0], [-2.0, 1.0], [1.0, 2.9]])
    s = O.fix_column_signs(u)
    assert np.array_equal(s[:, 0], -u[:, 0]) and np.array_equal(s[:, 1], -u[:, 1])
    tie = np.array([[-1.0], [1.0]])  # first max wins on ties
    assert np.array_equal(O.fix_column_signs(tie), -tie)


# ------------------------------------------------------------------ tucker.hpp
def test_rand_tucker_exact_rank_deterministic(O):  # test_tucker.cpp:96-106
    y = low_mlrank(O, (30, 30, 30), (5, 5, 5), 30)
    g, us = O.rand_tucker(y, (5, 5, 5), 10, (31, 0))
    assert O.fit(y, O.reconstruct(g, us)) > 1 - 1e-8
    assert all(orthonormality_defect(u) < 1e-10 for u in us)
    g2, us2 = O.rand_tucker(y, (5, 5, 5), 10, (31, 0))
    assert np.array_equal(g, g2) and all(np.array_equal(a, b) for a, b in zip(us, us2))


def test_rand_tucker_2i_exact_rank_deterministic(O):  # test_tucker.cpp:108-117
    y = low_mlrank(O, (30, 30, 30), (5, 5, 5), 32)
    g, us = O.rand_tucker_2i(y, (5, 5, 5), 10, (33, 0))
    assert O.fit(y, O.reconstruct(g, us)) > 1 - 1e-8
    assert all(orthonormality_defect(u) < 1e-10 for u in us)
    assert [u.shape[1] for u in us] == [5, 5, 5]  # rank cut drops the 10 oversampled columns
    g2, _ = O.rand_tucker_2i(y, (5, 5, 5), 10, (33, 0))
    assert np.array_equal(g, g2)


def test_two_pass_tracks_one_pass(O):  # test_tucker.cpp:119-134
    worst = 0.0
    for s in range(10):
        clean = low_mlrank(O, (24, 24, 24), (5, 5, 5), 100 + s)
        noise = rt(O, (24, 24, 24), 200 + s)
        y = clean + np.linalg.norm(clean) / np.linalg.norm(noise) * noise
        f1 = O.fit(y, O.reconstruct(*O.rand_tucker(y, (5, 5, 5), 10, (300 + s, 0))))
        f2 = O.fit(y, O.reconstruct(*O.rand_tucker_2i(y, (5, 5, 5), 10, (300 + s, 0))))
        worst = max(worst, f1 - f2)
    assert worst < 0.02


def test_reconstruct_identity(O):  # test_tucker.cpp:23-29
    core = rt(O, (3, 4, 2), 21)
    assert np.array_equal(O.reconstruct(core, [np.eye(3), np.eye(4), np.eye(2)]), core)


def test_core_equals_projection_of_x_last(O):
    """G = X_{N-1} x_{N-1} U_{N-1}^T (the identity the device path uses to skip pass 2N+1)."""
    clean = low_mlrank(O, (20, 18, 16), (4, 4, 4), 5)
    y = clean + 0.1 * rt(O, (20, 18, 16), 6)
    g, us = O.rand_tucker_2i(y, (4, 4, 4), 3, (7, 0))
    x = O.ttm_all(y, us, 2, True)
    g2 = O.ttm(x, us[2].T, 2)
    assert np.allclose(g, g2, rtol=1e-12, atol=1e-12)


def test_2i_steps_follow_reference_recipe(O):
    """Re-derives every (pass, n) step of Alg. 3 from the oracle's primitives."""
    y = low_mlrank(O, (12, 10, 9), (3, 3, 3), 40) + 0.05 * rt(O, (12, 10, 9), 41)
    seed = (42, 0)
    ranks, p = (3, 3, 3), 4
    g, us, zs = O.rand_tucker_2i(y, ranks, p, seed, return_sketches=True)
    fs = [O.gaussian_matrix(d, min(r + p, d), O.seed_derived(*seed, 0x0A3, n)) for n, (d, r) in enumerate(zip(y.shape, ranks))]
    k = 0
    for ps in range(2):
        for n in range(3):
            x = O.ttm_all(y, fs, n, True)
            om = O.gaussian_matrix(x.size // x.shape[n], min(ranks[n] + p, y.shape[n]), O.seed_derived(*seed, 0x0B3 + ps, n))
            z = O.unfold_times(x, n, om)
            assert np.allclose(z, zs[k], rtol=1e-13, atol=1e-13)
            fs[n] = O.fix_column_signs(O.orthonormal_basis(z))
            k += 1
    for a, b in zip(fs, us):
        assert np.allclose(a, b, rtol=1e-13, atol=1e-13)


# ------------------------------------------------------------------ ffcp.hpp
def test_ffcp_recovers_exact_cp(O):  # test_ffcp.cpp:90-96
    dims, R = (20, 20, 20, 20), 5
    fs = [O.gaussian_matrix(d, R, (77, 10 + n)) for n, d in enumerate(dims)]
    y = O.cp_reconstruct(fs)
    g, us = O.rand_tucker_2i(y, (5, 5, 5, 5), 10, (78, 0))
    a, trace, its = O.ffcp(g, us, 5, O.NONE, 0.0, 300, 1e-12, (79, 0))
    assert O.fit(y, O.cp_reconstruct(a)) > 1 - 1e-6


def _hosvd(y, ranks):
    us = []
    for n, r in enumerate(ranks):
        m = np.reshape(np.moveaxis(y, n, 0), (y.shape[n], -1), order="F")
        us.append(np.linalg.svd(m, full_matrices=False)[0][:, :r])
    return us


def test_ffcp_compressed_fit_equals_dense(O):  # test_ffcp.cpp:98-106
    y = low_mlrank(O, (10, 9, 8), (3, 3, 3), 80)
    us = _hosvd(y, (3, 3, 3))
    g = O.ttm_all(y, us, -1, True)
    a, trace, its = O.ffcp(g, us, 3, O.NONE, 0.0, 25, 0.0, (81, 0))
    assert its == 25
    yt = O.reconstruct(g, us)
    assert abs(trace[-1] - O.fit(yt, O.cp_reconstruct(a))) < 1e-8


def test_ffcp_nonneg_variants_stay_nonneg(O):  # test_ffcp.cpp:119-131
    fs = [np.abs(O.gaussian_matrix(d, 3, (84, n))) for n, d in enumerate((10, 9, 8))]
    y = O.cp_reconstruct(fs)
    g, us = O.rand_tucker_2i(y, (3, 3, 3), 5, (85, 0))
    for k in (1, 2, 4, 8):
        for kind in (O.NONNEG_MU, O.NONNEG_HALS):
            a, _, _ = O.ffcp(g, us, 3, kind, 0.0, k, 0.0, (86, 0))
            assert all(x.min() >= 0.0 for x in a)


def test_ffcp_hals_high_fit(O):  # test_ffcp.cpp:133-140
    fs = [np.abs(O.gaussian_matrix(15, 4, (87, n))) for n in range(3)]
    y = O.cp_reconstruct(fs)
    g, us = O.rand_tucker_2i(y, (4, 4, 4), 10, (88, 0))
    a, _, _ = O.ffcp(g, us, 4, O.NONNEG_HALS, 0.0, 400, 1e-12, (89, 0))
    assert O.fit(y, O.cp_reconstruct(a)) > 1 - 1e-4


def test_ffcp_sparse_zero_count_monotone(O):  # test_ffcp.cpp:142-153
    y = low_mlrank(O, (12, 12, 12), (4, 4, 4), 90)
    us = _hosvd(y, (4, 4, 4))
    g = O.ttm_all(y, us, -1, True)
    prev = -1
    for c in (0.0, 0.02, 0.05, 0.1, 0.3):
        a, _, _ = O.ffcp(g, us, 4, O.SPARSE, c, 30, 0.0, (91, 0))
        z = sum(int((x == 0.0).sum()) for x in a)
        assert z >= prev
        prev = z


def test_ffcp_rejects_bad_args(O):
    g = rt(O, (3, 3, 3), 1)
    us = [np.eye(3)] * 3
    with pytest.raises(ValueError, match="rank must be positive"):
        O.ffcp(g, us, 0)
    with pytest.raises(ValueError, match="sparsity"):
        O.ffcp(g, us, 2, O.SPARSE, -1.0)


# ------------------------------------------------------------------ generators (bench.hpp)
def test_generators_realised_snr(O):  # test_bench.cpp:37-53 (exact realised SNR)
    seed = (0, 5)
    y = O.gen_tucker((12, 11, 10), (3, 3, 3), seed)
    for snr in (0.0, 10.0, 20.0):
        for ab in (False, True):
            yn = O.add_noise(y, snr, seed, abs_noise=ab)
            e = yn - y
            real = 10 * np.log10(np.sum(y**2) / np.sum(e**2))
            assert abs(real - snr) < 1e-9
            if ab:
                assert (e >= 0).all()


def test_cp_uniform_generator(O):
    y, fs = O.gen_cp((6, 5, 4), 3, O.CP_UNIFORM, (1, 2))
    assert all(((a > 0) & (a <= 1)).all() for a in fs)
    ref = np.einsum("ir,jr,kr->ijk", *fs)
    assert np.allclose(y, ref, rtol=1e-14, atol=1e-14)
    # counter indexing mirrors bench.hpp:63-71: entry (i, j) of factor n at j*I_n + i
    fseed = O.seed_derived(1, 2, 0x9E4, 1)
    assert fs[1][3, 2] == O.uniform_at(fseed[0], fseed[1], 2 * 5 + 3)


# ------------------------------------------------------------------ streamed-slab oracle
@pytest.mark.parametrize("dims", [(30, 26, 22), (12, 10, 9, 8), (40, 33)])
@pytest.mark.parametrize("slab_elems", [1, 100, 1 << 30])
def test_streamed_oracle_matches_whole_tensor(O, dims, slab_elems):
    """The full-size checker (rand_tucker_2i over last-mode slabs of an fp32 host tensor,
    dist.hpp:496-596 pattern) equals the whole-tensor restatement on the same fp32 values:
    only the fp64 summation order over the last mode differs."""
    ranks = [3] * len(dims)
    y = O.add_noise(O.gen_tucker(dims, ranks, (0, 5)), 20.0, (0, 9))
    y32 = y.astype(np.float32)
    g, us = O.rand_tucker_2i(y32.astype(np.float64), ranks, 2, (1, 2))
    g2, us2, mg = O.rand_tucker_2i_streamed(y32.ravel(order="F"), dims, ranks, 2, (1, 2), slab_elems=slab_elems)
    for u, v in zip(us, us2):
        assert u.shape == v.shape and np.abs(u - v).max() < 1e-12
    assert np.abs(g - g2).max() < 1e-11 * np.abs(g).max()
    assert mg.shape == (2 * len(dims), 2) and np.all(mg >= 0) and np.all(mg <= 1)
