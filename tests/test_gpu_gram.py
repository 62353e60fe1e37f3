"""The distributed protocol's Gram-path orthonormalisation on the device (csrc/gram.cu) against
the oracle: gram_orthonormalize / gram_ortho_transform (range_finder.hpp:43-105) and the
numerics of dist_rand_tucker(_2i) (dist.hpp:688-723, 852-936), through the C-ABI.

The reference leaves each eigenvector's sign to Eigen's eigensolver and applies no sign rule
on this path, so factors are compared after aligning column signs (the core with the same
signs); eigenvalues, subspaces, the aligned factors/core and the fit are compared at the
north-star bars (1e-5 fp64, 1e-3 fp32; kernel level: fp64 rounding)."""
import os
import socket

import numpy as np
import pytest

from helpers import orthonormality_defect, subspace_dist

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


def signs(u, ref):
    s = np.sign(np.sum(u * ref, axis=0))
    s[s == 0] = 1.0
    return s


def align_core(g, ss):
    g = np.array(g, copy=True)
    for n, s in enumerate(ss):
        shape = [1] * g.ndim
        shape[n] = -1
        g = g * s.reshape(shape)
    return g


@pytest.mark.parametrize("rows,cols,nblocks", [(40, 5, 1), (40, 5, 2), (17, 3, 1), (1000, 30, 1), (1000, 30, 4),
                                               (4000, 60, 1), (200, 64, 1), (5000, 1, 3)])
def test_gram_orthonormalize_matches_oracle(P, O, rows, cols, nblocks):
    z = O.gaussian_matrix(rows, cols, (51, rows + cols))
    cuts = np.linspace(0, rows, nblocks + 1).astype(int)
    blocks = [z[a:b] for a, b in zip(cuts[:-1], cuts[1:])]
    u, sp = P.gram_orthonormalize(blocks)
    uo, spo = O.gram_orthonormalize(blocks)
    assert u.shape == uo.shape
    np.testing.assert_allclose(sp, spo, rtol=1e-12)
    assert orthonormality_defect(u) < 1e-12
    s = signs(u, uo)
    assert np.abs(u * s - uo).max() < 1e-10


def test_gram_orthonormalize_deficient_and_zero(P, O):
    base = O.gaussian_matrix(20, 2, (7, 0))
    z = np.column_stack([base[:, 0], base[:, 1], base[:, 0] + base[:, 1]])
    u, sp = P.gram_orthonormalize([z])
    assert u.shape == (20, 2) and sp.shape == (2,)
    assert subspace_dist(u, O.gram_orthonormalize([z])[0]) < 1e-10
    with pytest.raises(P.TenkitError, match="all blocks are zero"):
        P.gram_orthonormalize([np.zeros((4, 2)), np.zeros((6, 2))])


def test_gram_ortho_transform_matches_oracle(P, O):
    for n in (1, 2, 6, 31, 64):
        z = O.gaussian_matrix(3 * n + 4, n, (52, n))
        g = z.T @ z
        t, sp = P.gram_ortho_transform(g)
        to, spo = O.gram_ortho_transform(g)
        np.testing.assert_allclose(sp, spo, rtol=1e-12)
        assert orthonormality_defect(z @ t) < 1e-11
        assert np.abs(t * signs(t, to) - to).max() < 1e-9 * np.abs(to).max()


def _tensor(O, dims, ranks, seed, snr=20.0):
    y = O.gen_tucker(dims, ranks, seed)
    return O.add_noise(y, snr, O.seed_derived(*seed, 0xAD0))


@pytest.mark.parametrize("alg", ["2i", "alg2"])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("dims,ranks,p", [((60, 50, 40), (5, 5, 5), 5), ((300, 280, 260), (20, 20, 20), 10),
                                          ((24, 22, 20, 18), (4, 4, 4, 4), 3)])
def test_rand_tucker_gram_matches_oracle(P, O, alg, dtype, dims, ranks, p):
    """rand_tucker(_2i)(orthonormalizer='gram') == the oracle's dist_rand_tucker(_2i) numerics."""
    y = _tensor(O, dims, ranks, (61, len(dims))).astype(dtype)
    yd = P.DenseTensor.from_numpy(y, dtype).cuda()
    fn = P.rand_tucker_2i if alg == "2i" else P.rand_tucker
    m = fn(yd, list(ranks), p, (62, 1), orthonormalizer="gram").to_host()
    g_ref, u_ref = O.dist_rand_tucker_gram(y.astype(np.float64), list(ranks), p, (62, 1), alg=3 if alg == "2i" else 2)
    tol = F64_TOL if dtype == np.float64 else F32_TOL
    # fp32: the oversampled columns span noise whose Gram eigenvalues nearly coincide, so
    # fp32-level perturbations rotate those eigenvectors freely (an ill-posed comparison the
    # reference's own dist path has too); fp32 is compared on the leading R (signal) columns,
    # the matching core block and the fit. fp64: every column. Alg. 3 in fp32 feeds those
    # freely rotated noise columns into the second pass's sketch, so even its signal subspace
    # then differs by the randomized estimate's own statistical error (noise/signal ~ 0.1 at
    # 20 dB, measured 0.047): there only the fit is held to the 1e-3 bar.
    lead = [u.shape[1] if dtype == np.float64 else r for u, r in zip(u_ref, ranks)]
    sub_tol = 0.1 if (dtype == np.float32 and alg == "2i") else tol
    ss = []
    for u, uo, k in zip(m.factors, u_ref, lead):
        assert u.shape == uo.shape
        assert orthonormality_defect(u) < 1e-10
        assert subspace_dist(u[:, :k], uo[:, :k]) < sub_tol
        ss.append(signs(u, uo))
        if dtype == np.float64:
            assert np.abs(u * ss[-1] - uo).max() < 1e-8
    g = align_core(m.core, ss)[tuple(slice(0, k) for k in lead)]
    gr = g_ref[tuple(slice(0, k) for k in lead)]
    assert np.linalg.norm(g - gr) <= max(tol, sub_tol) * np.linalg.norm(gr)
    f = O.fit(y.astype(np.float64), O.reconstruct(m.core, m.factors))
    f_ref = O.fit(y.astype(np.float64), O.reconstruct(g_ref, u_ref))
    assert abs(f - f_ref) <= tol * abs(f_ref)


@pytest.mark.parametrize("dims,ranks,p", [((60, 50, 40), (5, 5, 5), 5), ((300, 280, 260), (20, 20, 20), 10)])
def test_gram_fp32_data_fp64_mode_matches_oracle_on_every_column(P, O, dims, ranks, p):
    """fp32 data on the distributed protocol's basis: in fp32 arithmetic the oversampled (noise)
    eigenvectors rotate freely (test above); precision='fp64' (fp64 arithmetic over the same
    fp32 values, the reference's own precision) reproduces the oracle's dist_rand_tucker_2i on
    EVERY r~ column up to eigenvector signs, the aligned core and the fit at the fp64 bar."""
    y = _tensor(O, dims, ranks, (61, len(dims))).astype(np.float32)
    yd = P.DenseTensor.from_numpy(y, np.float32).cuda()
    m = P.rand_tucker_2i(yd, list(ranks), p, (62, 1), orthonormalizer="gram", precision="fp64").to_host()
    g_ref, u_ref = O.dist_rand_tucker_gram(y.astype(np.float64), list(ranks), p, (62, 1), alg=3)
    ss = []
    for u, uo in zip(m.factors, u_ref):
        assert u.shape == uo.shape
        assert orthonormality_defect(u) < 1e-10
        assert subspace_dist(u, uo) < 1e-7
        ss.append(signs(u, uo))
        assert np.abs(u * ss[-1] - uo).max() < 1e-6
    g = align_core(m.core, ss)
    assert np.linalg.norm(g - g_ref) <= 1e-7 * np.linalg.norm(g_ref)
    f = O.fit(y.astype(np.float64), O.reconstruct(m.core, m.factors))
    f_ref = O.fit(y.astype(np.float64), O.reconstruct(g_ref, u_ref))
    assert abs(f - f_ref) <= 1e-9


def test_gram_rank_drop_and_replay(P, O):
    """Exact-rank data: the Gram cut (eigenvalues <= 1e-12 top) drops directions like the
    reference's dist path; repeated calls replay the captured graph identically; the
    context's default basis (ColPiv + sign rule) is restored afterwards."""
    from test_oracle_tucker import low_mlrank
    y = low_mlrank(O, (40, 40, 40), (5, 5, 5), 133)
    yd = P.DenseTensor.from_numpy(y).cuda()
    m = P.rand_tucker_2i(yd, [5, 5, 5], 10, (134, 0), orthonormalizer="gram").to_host()
    g_ref, u_ref = O.dist_rand_tucker_gram(y, [5, 5, 5], 10, (134, 0), alg=3)
    assert [u.shape[1] for u in m.factors] == [u.shape[1] for u in u_ref]
    assert O.fit(y, O.reconstruct(m.core, m.factors)) > 1.0 - 1e-8
    y2 = _tensor(O, (64, 60, 56), (6, 6, 6), (71, 0))
    y2d = P.DenseTensor.from_numpy(y2).cuda()
    ms = [P.rand_tucker_2i(y2d, [6, 6, 6], 4, (72, 0), orthonormalizer="gram").to_host() for _ in range(4)]
    for mm in ms[1:]:
        np.testing.assert_array_equal(mm.core, ms[0].core)
        for a, b in zip(mm.factors, ms[0].factors):
            np.testing.assert_array_equal(a, b)
    c = P.rand_tucker_2i(y2d, [6, 6, 6], 4, (72, 0)).to_host()
    _, uc = O.rand_tucker_2i(y2, [6, 6, 6], 4, (72, 0))
    for u, uo in zip(c.factors, uc):
        assert np.abs(u - uo).max() < 1e-8  # ColPiv + sign rule again: equal without sign alignment
    with pytest.raises(P.TenkitError, match="orthonormalizer"):
        P.rand_tucker_2i(y2d, [6, 6, 6], 4, (72, 0), orthonormalizer="svd")


# ---------------------------------------------------------------- block grid, gloo ranks on one GPU
BDIMS = (40, 36, 30)
RANKS = [5, 5, 5]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, grid, alg, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from oracle import pyoracle as O
        import paper_1412_1885_b200 as P
        from paper_1412_1885_b200.dist import GridPlan, MessageLog, dist_rand_tucker, dist_rand_tucker_2i
        O.build()
        y = _tensor(O, BDIMS, (5, 5, 5), (81, 0))
        log = MessageLog()
        plan = GridPlan.even(BDIMS, grid)
        lo, _ = plan.block(rank)
        ctx = P.Context.default()
        ctx.bind_torch_stream()
        yd = P.DenseTensor.from_numpy(plan.local(y, rank)).cuda()
        fn = dist_rand_tucker_2i if alg == "2i" else dist_rand_tucker
        m = fn(yd, BDIMS, lo, RANKS, 4, (82, 0), context=ctx, orthonormalizer="gram", log=log).to_host()
        counts = [log.count("partial_product", n) for n in range(3)] + [log.count("core_block")]
        q.put((rank, m.core, (m.factors, counts, [(r.rows, r.cols) for r in log.records()])))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported by the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc(), None))


@pytest.mark.parametrize("alg,grid", [("2i", (2, 2, 2)), ("alg2", (1, 2, 2))])
def test_block_grid_gram_protocol_matches_oracle(P, O, alg, grid):
    """dist_rand_tucker(_2i)(orthonormalizer='gram') over a BlockGrid: partial sketches summed
    over ranks, replicated Gram-eig basis — every rank holds the same model, equal to the
    oracle's dist_rand_tucker(_2i) numerics up to column signs."""
    import torch.multiprocessing as mp
    world = int(np.prod(grid))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, grid, alg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, core, extra = q.get(timeout=600)
        assert extra is not None, core
        fac, counts, shapes = extra
        # the exchange audit (MessageLog, dist.hpp:277-320): one Z all-reduce per range step, one core
        steps = 2 if alg == "2i" else 1
        assert counts == [steps, steps, steps, 1]
        assert shapes[-1][0] == int(np.prod(np.shape(core))) and all(c == 9 for _, c in shapes[:-1])
        res[r] = (core, fac)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = _tensor(O, BDIMS, (5, 5, 5), (81, 0))
    g_ref, u_ref = O.dist_rand_tucker_gram(y, RANKS, 4, (82, 0), alg=3 if alg == "2i" else 2)
    for r in range(world):
        core, fac = res[r]
        ss = []
        for u, uo in zip(fac, u_ref):
            ss.append(signs(u, uo))
            assert np.abs(u * ss[-1] - uo).max() < 1e-8
        g = align_core(core, ss)
        assert np.linalg.norm(g - g_ref) <= 1e-8 * np.linalg.norm(g_ref)
        for a, b in zip(res[0][1], fac):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(res[0][0], core)
