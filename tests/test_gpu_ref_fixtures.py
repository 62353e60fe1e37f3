"""The device path against the REFERENCE-RUN fixtures (tests/golden/ref_fixtures.npz: the
reference's own rand_tucker_2i / rand_tucker / orthonormal_basis executed from its unmodified
headers, tests/golden/make_ref_fixtures.py), through the C-ABI.

fp64 data: the north-star bar 1e-5 on subspaces / aligned core, and factor-by-factor 1e-8
(same pivot order, column signs and rank, incl. the rank-drop case); fp32 data on the device's
fp32 path: 1e-3 (the rank-drop case on its two real directions)."""
import numpy as np
import pytest

from helpers import subspace_dist

pytestmark = pytest.mark.gpu

FIX = __import__("os").path.join(__import__("os").path.dirname(__import__("os").path.abspath(__file__)), "golden",
                                 "ref_fixtures.npz")


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1412_1885_b200 as P
    return P


@pytest.fixture(scope="module")
def F():
    return np.load(FIX)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def _aligned(O, core, us, vs):
    return O.ttm_all(core, [u.T @ v for u, v in zip(us, vs)], -1, False)


@pytest.mark.parametrize("alg", ["2i", "a2"])
def test_fp64_device_matches_reference_run(P, O, F, alg):
    for name in [str(c) for c in F["cases"]]:
        key = f"{name}_f64"
        y, ranks, p = F[f"{key}_y"], [int(r) for r in F[f"{name}_ranks"]], int(F[f"{name}_p"])
        fn, seed = (P.rand_tucker_2i, (1, 2)) if alg == "2i" else (P.rand_tucker, (3, 4))
        m = fn(y, ranks, p, seed)
        refs = [F[f"{key}_{alg}_u{n}"] for n in range(len(ranks))]
        for u, v in zip(m.factors, refs):
            assert u.shape == v.shape, (name, u.shape, v.shape)  # incl. the reference's rank drop
            assert subspace_dist(u, v) < 1e-5
            assert np.abs(u - v).max() < 1e-8, name  # same pivots and signs
        g = F[f"{key}_{alg}_core"]
        assert rel(m.core, g) < 1e-8
        assert rel(_aligned(O, m.core, m.factors, refs), g) < 1e-5


def test_fp32_device_matches_reference_run(P, O, F):
    for name in [str(c) for c in F["cases"]]:
        key = f"{name}_f32"
        y, ranks, p = F[f"{key}_y"], [int(r) for r in F[f"{name}_ranks"]], int(F[f"{name}_p"])
        yd = P.DenseTensor.from_numpy(y.astype(np.float32), np.float32).cuda()
        m = P.rand_tucker_2i(yd, ranks, p, (1, 2), out="host")
        refs = [F[f"{key}_2i_u{n}"] for n in range(len(ranks))]
        for u, v in zip(m.factors, refs):
            assert u.shape == v.shape, (name, u.shape, v.shape)
            k = 2 if name == "rankdrop" else u.shape[1]  # fp32 rounding directions are not data
            assert subspace_dist(u[:, :k], v[:, :k]) < 1e-3, name
        if name != "rankdrop":
            assert rel(_aligned(O, m.core, m.factors, refs), F[f"{key}_2i_core"]) < 1e-3


def test_device_orthonormal_basis_matches_reference_run(P, F):
    for zk, uk in (("qr_z", "qr_u"), ("qr_z2", "qr_u2")):
        u = P.orthonormal_basis(F[zk])
        assert u.shape == F[uk].shape
        assert np.abs(u - F[uk]).max() < 1e-10
