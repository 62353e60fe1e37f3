"""The multi-GPU path through the C-ABI (slab-partitioned Y, tk_comm reduction hook) with
two ranks. Only one GPU is available to this run, so both ranks share cuda:0 over gloo
(host-staged all-reduce: no kernel of one rank waits on the other's); on a multi-GPU box
bench.py runs the same code over NCCL, one rank per GPU. The distributed model must equal
the single-process model of the whole tensor (dist.hpp:617-800 semantics: partial
sketches and cores summed over ranks, replicated QR) and the oracle."""
import os
import socket

import numpy as np
import pytest

from helpers import orthonormality_defect, subspace_dist

pytestmark = pytest.mark.gpu

DIMS, RANKS, P_OVER, SEED = (40, 36, 30), (4, 4, 4), 3, (7, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _tensor(O):
    data = O.seed_derived(3, 0, 0xDA7A)
    return O.add_noise(O.gen_tucker(DIMS, RANKS, data), 15.0, O.seed_derived(*data, 0xAD0))


def _worker(rank, world, port, sync, dtype, q, alg="2i"):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from oracle import pyoracle as O
        import paper_1412_1885_b200 as P
        from paper_1412_1885_b200.dist import dist_rand_tucker, dist_rand_tucker_2i, plan_slabs
        O.build()
        y = _tensor(O)
        off, ln = plan_slabs(DIMS[-1], world)[rank]
        yl = np.asfortranarray(y[:, :, off:off + ln]).astype(dtype)
        ctx = P.Context.default()
        ctx.bind_torch_stream()
        yd = P.DenseTensor.from_numpy(yl, dtype).cuda()
        if alg == "2i":
            m = dist_rand_tucker_2i(yd, DIMS[-1], off, RANKS, P_OVER, SEED, context=ctx, sync_ranks=sync).to_host()
        else:
            m = dist_rand_tucker(yd, DIMS[-1], off, RANKS, P_OVER, SEED, context=ctx).to_host()
        q.put((rank, m.core, m.factors, m.stats.get("passes")))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported by the parent
        q.put((rank, repr(e), None, None))


@pytest.mark.parametrize("sync", [True, False])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_two_rank_slabs_match_single_process(O, sync, dtype):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    import paper_1412_1885_b200 as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sync, dtype, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, core, fac, passes = q.get(timeout=300)
        assert fac is not None, core
        res[r] = (core, fac, passes)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = _tensor(O)
    single = P.rand_tucker_2i(P.DenseTensor.from_numpy(y.astype(dtype), dtype).cuda(), RANKS, P_OVER, SEED).to_host()
    g_ref, u_ref = O.rand_tucker_2i(y.astype(dtype).astype(np.float64), RANKS, P_OVER, SEED)
    tol = 1e-10 if dtype == np.float64 else 1e-4
    for r in (0, 1):
        core, fac, _ = res[r]
        for u, us, uo in zip(fac, single.factors, u_ref):
            assert orthonormality_defect(u) < 1e-10
            assert subspace_dist(u, us) < tol
            assert subspace_dist(u, uo) < (1e-8 if dtype == np.float64 else 1e-3)
        np.testing.assert_allclose(core, single.core, rtol=0, atol=tol * np.abs(single.core).max())
    # replicated QR: both ranks hold the identical model
    for a, b in zip(res[0][1], res[1][1]):
        np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(res[0][0], res[1][0])


def test_gaussian_fill_windows():
    """tk_gaussian_fill = a window of the flat counter stream at any (odd/even) offset."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1412_1885_b200 import SeedSpec
    from paper_1412_1885_b200.generators import gaussian_flat
    s = SeedSpec(9, 4)
    full = gaussian_flat(1001, s).cpu().numpy()
    for off, n in [(1, 10), (2, 999), (7, 1), (500, 501), (999, 2)]:
        np.testing.assert_array_equal(gaussian_flat(n, s, offset=off).cpu().numpy(), full[off:off + n])


def _gen_worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_1412_1885_b200.dist import plan_slabs
        from paper_1412_1885_b200.generators import generate

        def all_sum(x):
            t = torch.tensor([x], dtype=torch.float64)
            dist.all_reduce(t)
            return float(t.item())

        cfg = dict(dims=(24, 20, 31), gen="tucker", mlrank=(3, 4, 2), snr=20.0)
        off, ln = plan_slabs(31, world)[rank]
        y = generate(cfg, slab=(off, ln), all_sum=all_sum)
        q.put((rank, y.cpu().numpy()))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_blockwise_generation_concatenates_to_the_global_tensor():
    """generate(slab=...) on 2 ranks == generate() of the whole tensor (bench.hpp:83-112
    drawn at global indices), the data layout bench.py --gpus N uses."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    from paper_1412_1885_b200.generators import generate
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gen_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    assert all(isinstance(v, np.ndarray) for v in got.values()), got
    full = generate(dict(dims=(24, 20, 31), gen="tucker", mlrank=(3, 4, 2), snr=20.0)).cpu().numpy()
    cat = np.concatenate([got[0], got[1]])
    np.testing.assert_allclose(cat, full, rtol=0, atol=1e-12 * np.abs(full).max())


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_two_rank_alg2_matches_single_process(O, dtype):
    """dist_rand_tucker (Alg. 2) over two slabs == rand_tucker of the whole tensor == oracle."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    import paper_1412_1885_b200 as P
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, True, dtype, q, "alg2")) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, core, fac, _ = q.get(timeout=300)
        assert fac is not None, core
        res[r] = (core, fac)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = _tensor(O)
    single = P.rand_tucker(P.DenseTensor.from_numpy(y.astype(dtype), dtype).cuda(), RANKS, P_OVER, SEED).to_host()
    g_ref, u_ref = O.rand_tucker(y.astype(dtype).astype(np.float64), RANKS, P_OVER, SEED)
    tol = 1e-10 if dtype == np.float64 else 1e-4
    for r in (0, 1):
        core, fac = res[r]
        for u, us, uo in zip(fac, single.factors, u_ref):
            assert orthonormality_defect(u) < 1e-10
            assert subspace_dist(u, us) < tol
            assert subspace_dist(u, uo) < (1e-8 if dtype == np.float64 else 1e-3)
        np.testing.assert_allclose(core, single.core, rtol=0, atol=tol * np.abs(single.core).max())


# ---------------------------------------------------------------- general block grids
BDIMS = (40, 36, 30)


def _block_worker(rank, world, port, grid, alg, dtype, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from oracle import pyoracle as O
        import paper_1412_1885_b200 as P
        from paper_1412_1885_b200.dist import GridPlan, dist_rand_tucker, dist_rand_tucker_2i
        O.build()
        y = _tensor(O)
        plan = GridPlan.even(BDIMS, grid)
        lo, ln = plan.block(rank)
        ctx = P.Context.default()
        ctx.bind_torch_stream()
        yd = P.DenseTensor.from_numpy(plan.local(y, rank).astype(dtype), dtype).cuda()
        fn = dist_rand_tucker_2i if alg == "2i" else dist_rand_tucker
        m = fn(yd, BDIMS, lo, RANKS, P_OVER, SEED, context=ctx).to_host()
        q.put((rank, m.core, m.factors))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported by the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc(), None))


@pytest.mark.parametrize("alg,grid,dtype", [("2i", (2, 2, 2), np.float64), ("2i", (2, 2, 2), np.float32),
                                            ("2i", (1, 3, 1), np.float64), ("alg2", (2, 2, 2), np.float64),
                                            ("alg2", (3, 1, 2), np.float32)])
def test_block_grid_matches_single_process(O, alg, grid, dtype):
    """dist_rand_tucker(_2i) over a general BlockGrid (dist.hpp:24-123, e.g. BASELINE cfg 5's
    2 x 2 x 2 grid on 8 ranks): every rank projects its block with its rows of every factor,
    partial sketches (own rows of Z for partitioned modes) and partial cores are summed — the
    model equals the single-process model and the oracle; all ranks hold the identical model."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    import paper_1412_1885_b200 as P
    world = int(np.prod(grid))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_block_worker, args=(r, world, port, grid, alg, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, core, fac = q.get(timeout=600)
        assert fac is not None, core
        res[r] = (core, fac)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = _tensor(O)
    yt = P.DenseTensor.from_numpy(y.astype(dtype), dtype).cuda()
    if alg == "2i":
        single = P.rand_tucker_2i(yt, RANKS, P_OVER, SEED).to_host()
        g_ref, u_ref = O.rand_tucker_2i(y.astype(dtype).astype(np.float64), RANKS, P_OVER, SEED)
    else:
        single = P.rand_tucker(yt, RANKS, P_OVER, SEED).to_host()
        g_ref, u_ref = O.rand_tucker(y.astype(dtype).astype(np.float64), RANKS, P_OVER, SEED)
    tol = 1e-10 if dtype == np.float64 else 1e-4
    for r in range(world):
        core, fac = res[r]
        for u, us, uo in zip(fac, single.factors, u_ref):
            assert orthonormality_defect(u) < 1e-10
            assert subspace_dist(u, us) < tol
            assert subspace_dist(u, uo) < (1e-8 if dtype == np.float64 else 1e-3)
        np.testing.assert_allclose(core, single.core, rtol=0, atol=tol * np.abs(single.core).max())
        for a, b in zip(res[0][1], fac):  # replicated QR: identical models on every rank
            np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(res[0][0], core)


def test_block_generation_tiles_the_global_tensor():
    """generate_as(block=...) of every block of a 2 x 2 x 2 grid, placed at its offsets,
    == generate() of the whole tensor (every entry drawn at its global index; the sigma of
    the noise from norms summed over the blocks) — cfg 5's blockwise on-device generation."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1412_1885_b200.dist import GridPlan
    from paper_1412_1885_b200.generators import generate, generate_as, gaussian_block, gaussian_flat
    from paper_1412_1885_b200 import SeedSpec
    dims = (24, 20, 31)
    cfg = dict(dims=dims, gen="tucker", mlrank=(3, 4, 2), snr=20.0)
    full = generate(cfg).cpu().numpy().reshape(dims, order="F")
    plan = GridPlan.even(dims, (2, 2, 2))
    # noise/raw draws: the block fill equals the slice of the flat stream
    s = SeedSpec(4, 2)
    flat = gaussian_flat(int(np.prod(dims)), s).cpu().numpy().reshape(dims, order="F")
    for r in range(plan.world):
        lo, ln = plan.block(r)
        got = gaussian_block(dims, lo, ln, s).cpu().numpy().reshape(ln, order="F")
        np.testing.assert_array_equal(got, plan.local(flat, r))
    # sigma from the whole tensor's norms: sum the blocks' squared norms like all_sum would
    parts = {}
    # all_sum stand-in: first collect each block's (||Y||^2, ||E||^2), then feed the totals
    norms = []
    for r in range(plan.world):
        rec = []
        generate_as(cfg, torch.float64, block=plan.block(r), all_sum=lambda x, rec=rec: rec.append(x) or x)
        norms.append(rec)
    tot = [sum(v[i] for v in norms) for i in range(2)]
    for r in range(plan.world):
        it = iter(tot)
        parts[r] = generate_as(cfg, torch.float64, block=plan.block(r), all_sum=lambda x, it=it: next(it))
    out = np.zeros(dims)
    for r in range(plan.world):
        lo, ln = plan.block(r)
        out[lo[0]:lo[0] + ln[0], lo[1]:lo[1] + ln[1], lo[2]:lo[2] + ln[2]] = \
            parts[r].cpu().numpy().reshape(ln, order="F")
    np.testing.assert_allclose(out, full, rtol=0, atol=1e-12 * np.abs(full).max())


# ---------------------------------------------------------------- dist_multiply
def test_dist_multiply_single_block_equals_direct_product(O):
    """dist_multiply on a single block equals unfold(Y, n) * gaussian_matrix(width, r, seed)
    (reference test_dist.cpp:114-121), every mode, fp64 and fp32; reference error messages."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1412_1885_b200 as P
    from paper_1412_1885_b200.dist import dist_multiply
    y = O.gaussian_matrix(6 * 5 * 4, 1, (127, 0)).reshape((6, 5, 4), order="F")
    for dtype, tol in [(np.float64, 1e-10), (np.float32, 1e-5)]:
        yd = P.DenseTensor.from_numpy(y.astype(dtype), dtype).cuda()
        for mode in range(3):
            (z,) = dist_multiply(yd, (6, 5, 4), (0, 0, 0), mode, 3, (128, 0))
            om = O.gaussian_matrix(y.size // y.shape[mode], 3, (128, 0))
            direct = O.unfold_times(y.astype(dtype).astype(np.float64), mode, om)
            assert np.abs(z - direct).max() <= tol * np.abs(direct).max()
    with pytest.raises(P.TenkitError, match="r_tilde must be positive"):
        dist_multiply(yd, (6, 5, 4), (0, 0, 0), 0, 0, (1, 0))
    with pytest.raises(P.TenkitError, match="mode out of range"):
        dist_multiply(yd, (6, 5, 4), (0, 0, 0), 3, 2, (1, 0))


def _dm_worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from oracle import pyoracle as O
        import paper_1412_1885_b200 as P
        from paper_1412_1885_b200.dist import GridPlan, dist_multiply
        y = O.gaussian_matrix(8 * 6 * 3, 1, (129, 0)).reshape((8, 6, 3), order="F")
        plan = GridPlan((8, 6, 3), [[4, 4], [3, 3], [3]])
        lo, ln = plan.block(rank)
        yd = P.DenseTensor.from_numpy(plan.local(y, rank)).cuda()
        out = [dist_multiply(yd, (8, 6, 3), lo, mode, 4, (130, 0), grid=plan) for mode in range(3)]
        q.put((rank, out))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))


def test_dist_multiply_grid_matches_single_node(O):
    """dist_multiply across a 2 x 2 x 1 grid (4 ranks sharing cuda:0 over gloo): the stacked
    row blocks equal the single-node unfold(Y, n) * Omega (reference test_dist.cpp:123-139), for
    every mode; every rank holds the same blocks."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dm_worker, args=(r, 4, port, q)) for r in range(4)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(4))
    for p in procs:
        p.join(timeout=60)
    y = O.gaussian_matrix(8 * 6 * 3, 1, (129, 0)).reshape((8, 6, 3), order="F")
    for r in range(4):
        assert not isinstance(res[r], str), res[r]
        for mode in range(3):
            blocks = res[r][mode]
            assert len(blocks) == [2, 2, 1][mode]
            om = O.gaussian_matrix(y.size // y.shape[mode], 4, (130, 0))
            direct = O.unfold_times(y, mode, om)
            stacked = np.vstack(blocks)
            assert np.abs(stacked - direct).max() <= 1e-10 * np.abs(direct).max()
            for a, b in zip(blocks, res[0][mode]):
                np.testing.assert_array_equal(a, b)
