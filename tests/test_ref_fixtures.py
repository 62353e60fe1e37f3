"""The oracle against the REFERENCE-RUN fixtures (tests/golden/ref_fixtures.npz, made by
tests/golden/make_ref_fixtures.py from the reference's own tensor/random/range_finder/
tucker.hpp compiled unmodified against oracle/ref_shim): this pins the oracle's hot-path
numerics — counter RNG, seed tags, ttm / unfold_times, the pivoted QR + sign rule and the
rand_tucker_2i / rand_tucker control flow, incl. rank drop — to the reference's execution,
not to a second restatement. Where oracle/_ref is built (this container) the oracle is also
compared live on fresh seeds."""
import os

import numpy as np
import pytest

FIX = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_fixtures.npz")


@pytest.fixture(scope="module")
def F():
    return np.load(FIX)


def _close(a, b, tol):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    scale = max(1.0, float(np.abs(b).max()) if b.size else 1.0)
    assert float(np.abs(a - b).max() if a.size else 0.0) <= tol * scale


def test_rng_matches_reference_run(O, F):
    for s, ref in zip(F["rng_seeds"], F["rng_normals"]):
        got = O.gaussian_matrix(9, 3, (int(s[0]), int(s[1]))).ravel(order="F")
        np.testing.assert_array_equal(got, ref)  # bit-exact (same libm transcendental kernels)
    tags = (0x0A2, 0x0A3, 0x0B3, 0x0B4, 0xC0DE)
    assert [O.seed_derived(33, 0, t)[1] for t in tags] == [int(x) for x in F["rng_derived"]]


def test_kernels_match_reference_run(O, F):
    t = F["k_t"]
    for n in range(3):
        _close(O.ttm(t, F[f"k_ttm_m{n}"], n), F[f"k_ttm_out{n}"], 1e-13)
        _close(O.unfold_times(t, n, F[f"k_ut_b{n}"]), F[f"k_ut_out{n}"], 1e-13)


@pytest.mark.parametrize("zk,uk", [("qr_z", "qr_u"), ("qr_z2", "qr_u2")])
def test_orthonormal_basis_matches_reference_run(O, F, zk, uk):
    u = O.fix_column_signs(O.orthonormal_basis(F[zk]))
    _close(u, F[uk], 1e-12)  # same rank, pivot order and column signs


def _cases(F):
    return [str(c) for c in F["cases"]]


@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_decompositions_match_reference_run(O, F, tag):
    for name in _cases(F):
        key = f"{name}_{tag}"
        y, ranks, p = F[f"{key}_y"], [int(r) for r in F[f"{name}_ranks"]], int(F[f"{name}_p"])
        # exact rank-2 data rounded to fp32 keeps directions of relative size ~1e-8 above the
        # 1e-12 rank cut: those columns are conditioned at ~eps / 1e-8 (either QR implementation)
        tol = 1e-5 if (name == "rankdrop" and tag == "f32") else 1e-10
        g, us = O.rand_tucker_2i(y, ranks, p, (1, 2))
        _close(g, F[f"{key}_2i_core"], tol)
        for n, u in enumerate(us):
            _close(u, F[f"{key}_2i_u{n}"], tol)  # factor by factor: same pivots, signs, rank
        g, us = O.rand_tucker(y, ranks, p, (3, 4))
        _close(g, F[f"{key}_a2_core"], tol)
        for n, u in enumerate(us):
            _close(u, F[f"{key}_a2_u{n}"], tol)


def test_oracle_matches_live_reference_on_fresh_seeds(O):
    """Only where the reference sources are present (oracle/_ref built from them)."""
    if not os.path.isdir("/root/reference/proj/include/tenkit"):
        pytest.skip("reference sources absent (GPU box): the committed fixtures stand in")
    for k, (dims, ranks, p) in enumerate([((17, 15, 13), (3, 4, 2), 2), ((9, 8, 7, 6), (2, 3, 2, 2), 2),
                                          ((31, 12), (4, 4), 3)]):
        y = O.ref_gaussian_matrix(int(np.prod(dims)), 1, (900 + k, 1)).reshape(dims, order="F")
        g_ref, u_ref = O.ref_rand_tucker_2i(y, ranks, p, (k, 77))
        g, us = O.rand_tucker_2i(y, ranks, p, (k, 77))
        _close(g, g_ref, 1e-10)
        for u, v in zip(us, u_ref):
            _close(u, v, 1e-10)
        z = O.ref_gaussian_matrix(60, 9, (k, 5))
        _close(O.fix_column_signs(O.orthonormal_basis(z)), O.ref_orthonormal_basis(z), 1e-12)
