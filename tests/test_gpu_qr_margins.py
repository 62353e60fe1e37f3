"""The QR's discrete choices under near ties (SURVEY §7 hard part 1): the column pivot of
orthonormal_basis (range_finder.hpp:18-29) and the sign rule (tucker.hpp:39-45).

The device's fast path pivots on the Schur diagonals of a pivoted Cholesky of Z^T Z, whose
cancellation error is larger than the Householder norm downdate the reference (and the oracle)
use; when the two best pivot candidates are within the near-tie gap (1e-6 relative in squared
norms) the kernel falls back to the Householder path. Checked here: constructed near-tie Z's
take the fallback and match the oracle's pivots and factors; the reported pivot / sign margins
match the oracle's diagnostics; decompositions report per-step margins and QR paths."""
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


def _q(O, rows, cols, seed):
    q, _ = np.linalg.qr(O.gaussian_matrix(rows, cols, (seed, 1)))
    return q


def _near_tie_z(O, gap, step, rows=400, cols=12, seed=3):
    """Z = Q R0 with R0 upper triangular chosen so that at pivot step `step` the two largest
    remaining column norms differ by `gap` (relative) while every other choice is clear."""
    rng = np.random.default_rng(seed)
    r0 = np.zeros((cols, cols))
    norms = 10.0 * 0.7 ** np.arange(cols)  # clear pivot order by residual norm
    for j in range(cols):
        r0[j, j] = norms[j]
        r0[:j, j] = 0.01 * norms[j] * rng.standard_normal(j)  # small couplings
    # columns step and step+1: equal residual norms below row `step`, different couplings above
    a, b = step, step + 1
    r0[:, b] = 0.0
    r0[:a, b] = 0.5 * r0[:a, a] + 0.02 * norms[a]
    r0[a, b] = 0.6 * norms[a] * (1.0 + gap)
    r0[b, b] = 0.8 * norms[a] * (1.0 + gap)
    return _q(O, rows, cols, seed) @ r0


@pytest.mark.parametrize("step", [0, 1, 4])
@pytest.mark.parametrize("gap", [1e-9, 1e-8, 3e-8])
def test_near_tie_pivot_takes_householder_and_matches_oracle(P, O, step, gap):
    z = _near_tie_z(O, gap, step)
    u_ref, diag = O.orthonormal_basis(z, diagnostics=True)
    u_ref = O.fix_column_signs(u_ref)
    u, mg = P.orthonormal_basis(z, with_margins=True)
    assert mg["qr_path"] == 1  # the near tie sends the pivot decision to the Householder path
    assert u.shape == u_ref.shape
    assert np.abs(u - u_ref).max() < 1e-10  # same pivots (column order) and signs
    # the margin is the tie's gap: (top - second) / top in norms
    assert abs(mg["pivot_margin"] - diag["pivot_margin"][: z.shape[1] - 1].min()) < 1e-9


def test_clear_pivots_take_the_fast_path_with_oracle_margins(P, O):
    z = O.gaussian_matrix(1000, 30, (4, 4)) @ np.diag(1.0 + 0.05 * np.arange(30))
    u_ref, diag = O.orthonormal_basis(z, diagnostics=True)
    u_ref = O.fix_column_signs(u_ref)
    u, mg = P.orthonormal_basis(z, with_margins=True)
    assert np.abs(u - u_ref).max() < 1e-10
    pm = diag["pivot_margin"][: z.shape[1] - 1].min()
    if pm > 1e-5:
        assert mg["qr_path"] == 0
    assert abs(mg["pivot_margin"] - pm) < 1e-8 * max(1.0, pm)
    # sign margin: min over columns of (max |u| of the chosen sign - max of the other) / max
    top = np.abs(u_ref).max(axis=0)
    pos = np.where(u_ref > 0, u_ref, 0).max(axis=0)
    neg = np.where(u_ref < 0, -u_ref, 0).max(axis=0)
    assert abs(mg["sign_margin"] - float(np.min(np.abs(pos - neg) / top))) < 1e-10


def test_decomposition_reports_step_margins(P, O):
    seed = (2, 5)
    y = O.add_noise(O.gen_tucker((60, 50, 40), (4, 4, 4), seed), 20.0, O.seed_derived(*seed, 0xAD0))
    m = P.rand_tucker_2i(y, (4, 4, 4), 3, (1, 1))
    g_ref, u_ref, margins = O.rand_tucker_2i_streamed(y.astype(np.float32).ravel(order="F"), (60, 50, 40), (4, 4, 4), 3,
                                                      (1, 1))
    st = m.stats
    assert len(st["pivot_margin"]) == 6 and len(st["qr_path"]) == 6
    assert all(p in (0, 1) for p in st["qr_path"])
    # fp64 device run on fp64 Y vs the oracle on the fp32-rounded Y: margins agree loosely
    for k in range(6):
        assert 0.0 <= st["pivot_margin"][k] <= 1.0 and 0.0 <= st["sign_margin"][k] <= 1.0
    yd = P.DenseTensor.from_numpy(y.astype(np.float32), np.float32).cuda()
    m32 = P.rand_tucker_2i(yd, (4, 4, 4), 3, (1, 1), sync_ranks=False)
    for k in range(6):
        assert abs(m32.stats["pivot_margin"][k] - margins[k, 0]) < 1e-3
        assert abs(m32.stats["sign_margin"][k] - margins[k, 1]) < 1e-3


def test_device_path_limits_fail_loudly(P, O):
    """The documented device limit (include/tenkit_b200.h): r~ <= 64 raises the reference-style
    invalid_argument (TenkitError) instead of computing garbage. tk_qr_max_rows is the
    single-cluster capacity; taller sketches take the blocked path (tests below)."""
    import torch
    lib = P.Context.default().lib
    cap = int(lib.tk_qr_max_rows(60))
    assert 6000 < cap < 7000 and int(lib.tk_qr_max_rows(30)) > 2 * 6000 and int(lib.tk_qr_max_rows(65)) == 0
    y = torch.zeros(80 * 4 * 4, dtype=torch.float32, device="cuda")
    with pytest.raises(P.TenkitError, match="rank \\+ oversample must be <= 64"):
        P.rand_tucker_2i(P.DenseTensor((80, 4, 4), y), (60, 2, 2), 10, (0, 0))


@pytest.mark.parametrize("rows,cols", [(7000, 60), (20000, 60), (30000, 30), (60000, 64), (60000, 7)])
def test_tall_sketch_blocked_qr_matches_oracle(P, O, rows, cols):
    """Sketches taller than one cluster's shared memory (rows > tk_qr_max_rows): TSQR reduction
    of balanced row blocks, then the cluster ColPiv QR on the stacked R factors
    (range_finder.hpp:18-29 is invariant under the orthogonal reduction), sign rule on the
    product (tucker.hpp:39-45). Same pivots, |R_kk|, U and margins as the oracle."""
    lib = P.Context.default().lib
    assert rows > int(lib.tk_qr_max_rows(cols))
    z = O.gaussian_matrix(rows, cols, (rows, cols))
    if cols > 2:
        z[:, 1] = 3.0 * z[:, 0] + 1e-3 * z[:, 1]
    u_ref, d = O.orthonormal_basis(z, diagnostics=True)
    u_ref = O.fix_column_signs(u_ref)
    u, diag, mg = P.orthonormal_basis(z, with_diag=True, with_margins=True)
    assert u.shape == u_ref.shape
    assert np.allclose(np.abs(diag), np.abs(d["rdiag"]), rtol=1e-10, atol=1e-12)  # same pivots, same R_kk
    assert np.max(np.abs(u - u_ref)) < 1e-10
    assert np.linalg.norm(u.T @ u - np.eye(u.shape[1])) < 1e-12
    assert 0.0 < mg["pivot_margin"] <= 1.0 and 0.0 < mg["sign_margin"] <= 1.0


def test_tall_sketch_rank_deficient(P, O):
    """Blocked path with a rank-deficient sketch: the reduced matrix takes the Householder path
    and the rank cut drops the same columns as the oracle."""
    rows, cols, r = 9000, 48, 11
    z = O.gaussian_matrix(rows, r, (5, 0)) @ O.gaussian_matrix(r, cols, (5, 1))
    u_ref = O.fix_column_signs(O.orthonormal_basis(z))
    u, mg = P.orthonormal_basis(z, with_margins=True)
    assert u.shape == u_ref.shape == (rows, r) and mg["qr_path"] == 1
    assert np.linalg.norm(u @ u.T @ u_ref - u_ref) < 1e-9  # same subspace
    assert np.linalg.norm(u.T @ u - np.eye(r)) < 1e-12


def test_long_mode_decomposition_matches_oracle(P, O):
    """rand_tucker_2i with a mode longer than the cluster QR holds (20000 x 24 x 20, r~ = 60 in
    mode 0): fp64 factors / core / fit equal the oracle's (the reference accepts any shape)."""
    from test_gpu_parity import compare_models
    dims, ranks, p = (20000, 24, 20), (50, 6, 6), 10
    y = O.gen_tucker(dims, (8, 5, 5), (2, 0))
    y = O.add_noise(y, 25.0, (2, 1))
    ref = O.rand_tucker_2i(y, ranks, p, (7, 0))
    got = P.rand_tucker_2i(P.DenseTensor.from_numpy(y), ranks, p, (7, 0))
    compare_models(O, y, got, ref, 1e-8)
