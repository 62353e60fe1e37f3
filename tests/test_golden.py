"""Committed golden fixtures (tests/golden/oracle_golden.npz, made by tests/golden/make_golden.py).

CPU half: the oracle reproduces the fixtures (RNG bit-exact, numerics to 1e-12), so an
oracle regression cannot silently move the target the device is checked against.
GPU half: the device path, through the C-ABI, lands on the same fixtures within the
north_star tolerances (fp64 1e-5 on subspaces/core/fit)."""
import os

import numpy as np
import pytest

from helpers import np_key, np_normal, orthonormality_defect, subspace_dist

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_golden.npz"))


def close(a, b, tol=1e-12):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b))) <= tol * max(1.0, float(np.max(np.abs(b))))


def test_golden_rng(O):
    for s, key, normals, unif in zip(G["rng_seeds"], G["rng_keys"], G["rng_normals"], G["rng_uniforms"]):
        root, stream = int(s[0]), int(s[1])
        assert O.seed_key(root, stream) == int(key)
        assert int(np_key(root, stream)) == int(key)
        np.testing.assert_array_equal(O.gaussian_matrix(16, 1, (root, stream)).ravel(), normals)
        np.testing.assert_allclose(np_normal(int(key), np.arange(16, dtype=np.uint64)), normals, rtol=0, atol=1e-15)
        np.testing.assert_array_equal([O.uniform_at(root, stream, i) for i in range(16)], unif)
    assert [O.seed_derived(33, 0, 0x0A3, n)[1] for n in range(4)] == [int(v) for v in G["rng_derived"]]


def test_golden_qr(O):
    O.set_threads(1, use_blas=False)
    try:
        u, d = O.orthonormal_basis(G["qr_z"], diagnostics=True)
    finally:
        O.set_threads(1)
    assert u.shape == G["qr_u"].shape == (40, 6)
    np.testing.assert_array_equal(d["perm"], G["qr_perm"])
    assert close(O.fix_column_signs(u), G["qr_u"])
    assert close(d["rdiag"], G["qr_rdiag"])


def test_golden_tucker_and_ffcp(O):
    O.set_threads(1, use_blas=False)
    try:
        y = G["tucker_y"]
        data = O.seed_derived(0, 0, 0xDA7A, 0)
        y2 = O.add_noise(O.gen_tucker((20, 18, 16), (4, 4, 4), data), 10.0, O.seed_derived(*data, 0xAD0))
        assert close(y2, y)
        g, us = O.rand_tucker_2i(y, (4, 4, 4), 3, (7, 0))
        assert close(g, G["rt2i_core"], 1e-10)
        for n, u in enumerate(us):
            assert close(u, G[f"rt2i_u{n}"], 1e-10)
        g1, us1 = O.rand_tucker(y, (4, 4, 4), 3, (7, 0))
        assert close(g1, G["rt_core"], 1e-10)
        for n, u in enumerate(us1):
            assert close(u, G[f"rt_u{n}"], 1e-10)
        a, trace, _ = O.ffcp(g, us, 3, O.NONE, 0.0, 50, 1e-9, (8, 0))
        assert close(trace, G["ffcp_trace"], 1e-9)
    finally:
        O.set_threads(1)


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1412_1885_b200 as P
    return P


@pytest.mark.gpu
def test_golden_device_rng(P):
    for s, normals in zip(G["rng_seeds"], G["rng_normals"]):
        got = P.gaussian_matrix(16, 1, (int(s[0]), int(s[1])))
        np.testing.assert_allclose(np.asarray(got).ravel(), normals, rtol=0, atol=1e-14)


@pytest.mark.gpu
def test_golden_device_qr(P):
    u = P.orthonormal_basis(G["qr_z"])
    assert u.shape == (40, 6)
    assert orthonormality_defect(u) < 1e-12
    assert subspace_dist(u, G["qr_u"]) < 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("alg", ["rand_tucker_2i", "rand_tucker"])
def test_golden_device_tucker(P, alg):
    pre = "rt2i" if alg == "rand_tucker_2i" else "rt"
    y = P.DenseTensor.from_numpy(G["tucker_y"], np.float64).cuda()
    m = getattr(P, alg)(y, (4, 4, 4), 3, (7, 0)).to_host()
    for n, u in enumerate(m.factors):
        assert subspace_dist(u, G[f"{pre}_u{n}"]) < 1e-5
        np.testing.assert_allclose(u, G[f"{pre}_u{n}"], rtol=0, atol=1e-5)
    np.testing.assert_allclose(m.core, G[f"{pre}_core"], rtol=0, atol=1e-5 * np.abs(G[f"{pre}_core"]).max())


@pytest.mark.gpu
def test_golden_device_ffcp(P):
    model = P.TuckerModel(G["rt2i_core"], [G[f"rt2i_u{n}"] for n in range(3)], G["rt2i_core"].shape)
    res = P.ffcp(model, 3, P.ConstraintSpec(P.ConstraintKind.none), P.StopRule(50, 1e-9), (8, 0))
    n = min(len(res.fit_trace), len(G["ffcp_trace"]))
    np.testing.assert_allclose(res.fit_trace[:n], G["ffcp_trace"][:n], rtol=0, atol=1e-5)
