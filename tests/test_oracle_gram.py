"""Pins the oracle's Gram-path orthonormalisation (the reference's distributed protocol,
range_finder.hpp:43-105, dist.hpp:688-723, dist_rand_tucker(_2i) dist.hpp:852-936).

Mirrors test_range_finder.cpp:66-96 (gram_orthonormalize) and test_dist.cpp:141-152
(dist_rand_tucker == rand_tucker up to rotation), and pins the Jacobi eigensolver that stands
in for Eigen's SelfAdjointEigenSolver against LAPACK (numpy.linalg.eigh): eigenvalues to
rounding, eigenvectors up to sign."""
import numpy as np
import pytest

from helpers import max_principal_angle, orthonormality_defect
from test_oracle_tucker import low_mlrank


@pytest.mark.parametrize("n", [1, 2, 3, 7, 16, 30, 31, 60, 64])
def test_sym_eig_matches_lapack(O, n):
    z = O.gaussian_matrix(3 * n + 5, n, (41, n))
    g = z.T @ z
    ev, v = O.sym_eig(g)
    ev2, v2 = np.linalg.eigh(g)
    assert np.all(np.diff(ev) >= 0)  # ascending, Eigen's order
    assert np.max(np.abs(ev - ev2)) <= 1e-13 * ev2[-1]
    assert orthonormality_defect(v) < 1e-13
    np.testing.assert_allclose(np.abs(v.T @ v2), np.eye(n), atol=1e-9)  # distinct eigenvalues: same vectors up to sign
    assert np.linalg.norm(g @ v - v * ev) <= 1e-13 * ev2[-1] * n


def test_sym_eig_repeated_and_graded_spectra(O):
    g = np.eye(6) * 3.0  # repeated eigenvalue: any orthonormal basis, A V = V L
    ev, v = O.sym_eig(g)
    np.testing.assert_allclose(ev, 3.0, rtol=0, atol=1e-15)
    assert orthonormality_defect(v) < 1e-15
    z = O.gaussian_matrix(500, 30, (42, 0)) @ np.diag(np.logspace(0, -5, 30))  # cond(G) = 1e10
    g = z.T @ z
    ev, v = O.sym_eig(g)
    ev2 = np.linalg.eigvalsh(g)
    assert np.max(np.abs(ev - ev2) / ev2) < 1e-6  # Jacobi: relative accuracy on graded matrices
    assert np.linalg.norm(g @ v - v * ev) <= 1e-13 * ev2[-1] * 30


def test_gram_ortho_transform(O):
    z = O.gaussian_matrix(40, 6, (43, 0))
    t, sp = O.gram_ortho_transform(z.T @ z)
    assert t.shape == (6, 6) and sp.shape == (6,)
    assert np.all(np.diff(sp) <= 0)  # descending
    assert orthonormality_defect(z @ t) < 1e-12
    np.testing.assert_allclose(sp, np.linalg.eigvalsh(z.T @ z)[::-1], rtol=1e-13)
    with pytest.raises(O.OracleError, match="zero Gram matrix"):
        O.gram_ortho_transform(np.zeros((3, 3)))


def test_gram_orthonormalize_stacks_to_an_orthonormal_basis(O):  # test_range_finder.cpp:66-82
    z = O.gaussian_matrix(40, 5, (6, 0))
    q, _ = O.gram_orthonormalize([z])
    assert np.abs(q.T @ q - np.eye(5)).max() < 1e-10
    stacked, _ = O.gram_orthonormalize([z[:15], z[15:]])
    assert np.abs(stacked.T @ stacked - np.eye(stacked.shape[1])).max() < 1e-10
    assert max_principal_angle(O.orthonormal_basis(z), stacked) < 1e-8
    np.testing.assert_allclose(np.abs(stacked), np.abs(q), atol=1e-12)  # block split = rounding only


def test_gram_orthonormalize_rejects_all_zero_blocks(O):  # test_range_finder.cpp:84-87
    with pytest.raises(O.OracleError):
        O.gram_orthonormalize([np.zeros((4, 2)), np.zeros((6, 2))])


def test_gram_orthonormalize_drops_deficient_directions(O):  # test_range_finder.cpp:89-96
    base = O.gaussian_matrix(20, 2, (7, 0))
    z = np.column_stack([base[:, 0], base[:, 1], base[:, 0] + base[:, 1]])
    q, sp = O.gram_orthonormalize([z])
    assert q.shape[1] == 2 and sp.shape == (2,)


@pytest.mark.parametrize("alg", [2, 3])
def test_dist_gram_matches_single_node_up_to_rotation(O, alg):  # test_dist.cpp:141-152
    y = low_mlrank(O, (18, 16, 14), (4, 4, 4), 131)
    seed = (132, 0)
    g, us = O.dist_rand_tucker_gram(y, [4, 4, 4], 6, seed, alg=alg)
    gs, uss = (O.rand_tucker if alg == 2 else O.rand_tucker_2i)(y, [4, 4, 4], 6, seed)[:2]
    f_dist = O.fit(y, O.reconstruct(g, us))
    f_single = O.fit(y, O.reconstruct(gs, uss))
    assert abs(f_dist - f_single) < 1e-10
    for u, v in zip(uss, us):
        assert orthonormality_defect(v) < 1e-10
        assert max_principal_angle(u, v) < 1e-6


def test_dist_gram_recovers_exact_rank(O):  # test_dist.cpp:154-159
    y = low_mlrank(O, (40, 40, 40), (5, 5, 5), 133)
    g, us = O.dist_rand_tucker_gram(y, [5, 5, 5], 10, (134, 0), alg=2)
    assert O.fit(y, O.reconstruct(g, us)) > 1.0 - 1e-8
