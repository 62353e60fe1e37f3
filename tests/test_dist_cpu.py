"""Multi-rank path on CPU (gloo, world_size 2): the slab plan, the tk_comm reduction hook
(DistComm) and the sharding identity the device driver relies on —

  for n != N-1:  Z_n = sum_g unfold(Y^g x_{p != n} U_p^T, n) Omega_n   (rank g uses rows
                 [off_g, off_g + L_g) of U_{N-1})
  for n == N-1:  rank g owns rows [off_g, off_g + L_g) of Z_{N-1} (others zero-padded)
  core:          G = sum_g Y^g x_0 U_0^T ... x_{N-1} U_{N-1}[off_g:off_g+L_g]^T

(dist.hpp:617-800 semantics). Partial products come from the CPU oracle (test
infrastructure); the reduction goes through DistComm over torch.distributed/gloo."""
import os
import socket

import numpy as np
import pytest


def test_plan_slabs_matches_reference_partition():
    from paper_1412_1885_b200.dist import plan_slabs
    assert [l for _, l in plan_slabs(300, 8)] == [38, 38, 38, 38, 37, 37, 37, 37]
    for dim, w in [(1000, 1), (1000, 3), (7, 7), (4000, 8)]:
        sl = plan_slabs(dim, w)
        assert sum(l for _, l in sl) == dim and sl[0][0] == 0
        assert all(sl[i][0] + sl[i][1] == sl[i + 1][0] for i in range(w - 1))
        assert max(l for _, l in sl) - min(l for _, l in sl) <= 1
    from paper_1412_1885_b200 import TenkitError
    with pytest.raises(TenkitError, match="segment lengths must be positive"):
        plan_slabs(3, 4)


def test_exchange_capacity():
    from paper_1412_1885_b200.dist import exchange_capacity
    assert exchange_capacity((1000, 1000, 1000), (20, 20, 20), 10) == max(1000 * 30, 30 ** 3)
    assert exchange_capacity((100, 100, 100), (20, 20, 20), 10) == 30 ** 3
    assert exchange_capacity((4000, 10, 10), (5, 5, 5), 1) == 4000 * 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import pyoracle as O
        from paper_1412_1885_b200.dist import DistComm, plan_slabs, exchange_capacity
        O.set_threads(1)
        dims, ranks, p = (14, 12, 11), (3, 3, 3), 2
        seed = (5, 0)
        y = O.add_noise(O.gen_tucker(dims, ranks, seed), 10.0, O.seed_derived(*seed, 0xAD0))
        off, ln = plan_slabs(dims[-1], world)[rank]
        yl = np.asfortranarray(y[:, :, off:off + ln])
        rts = [min(r + p, i) for r, i in zip(ranks, dims)]
        us = [O.gaussian_matrix(i, r, (9, n)) for n, (i, r) in enumerate(zip(dims, rts))]
        comm = DistComm(off, dims[-1], exchange_capacity(dims, ranks, p))
        assert comm.world == world and comm.rank == rank
        errs = []
        for n in range(3):
            om = O.gaussian_matrix(int(np.prod([rts[k] for k in range(3) if k != n])), rts[n], (11, n))
            full = O.unfold_times(O.ttm_all(y, us, n, True), n, om)
            ul = [u if k != 2 else u[off:off + ln] for k, u in enumerate(us)]
            part = O.unfold_times(O.ttm_all(yl, ul, n, True), n, om)
            if n == 2:  # local rows of Z_{N-1}, zero-padded
                zp = np.zeros_like(full)
                zp[off:off + ln] = part
                part = zp
            comm.xbuf[: part.size] = __import__("torch").from_numpy(part.ravel(order="F"))
            assert comm.allreduce(part.size) == 0
            got = comm.xbuf[: part.size].numpy().reshape(full.shape, order="F")
            errs.append(float(np.abs(got - full).max() / np.abs(full).max()))
        g_full = O.ttm_all(y, us, -1, True)
        ul = [u if k != 2 else u[off:off + ln] for k, u in enumerate(us)]
        g_part = O.ttm_all(yl, ul, -1, True)
        comm.xbuf[: g_part.size] = __import__("torch").from_numpy(g_part.ravel(order="F"))
        comm.allreduce(g_part.size)
        g_got = comm.xbuf[: g_part.size].numpy().reshape(g_full.shape, order="F")
        errs.append(float(np.abs(g_got - g_full).max() / np.abs(g_full).max()))
        st = comm.as_struct()
        assert st.world == world and st.slab_offset == off and st.global_last_dim == dims[-1]
        q.put((rank, errs, comm.calls))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure in the parent
        import traceback
        q.put((rank, repr(e) + traceback.format_exc(), -1))


def test_gloo_world2_partial_sketches_reduce_to_single_node():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=180) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, errs, calls in res:
        assert calls == 4, errs
        assert max(errs) < 1e-12, errs


def test_grid_plan_mirrors_reference_partition():
    """GridPlan = partition/ind2sub/sub2ind (dist.hpp:45-123): worker ids are P = reshape(1..W)
    column-major over the grid, blocks tile the tensor exactly, errors carry the reference's
    messages. KAT: ind2sub((2,4,3), 13) = (1,3,2) (test_dist.cpp:32-40)."""
    from paper_1412_1885_b200 import TenkitError
    from paper_1412_1885_b200.dist import GridPlan, default_grid, ind2sub, sub2ind
    assert ind2sub([2, 4, 3], 13) == [1, 3, 2]
    assert sub2ind([2, 4, 3], [1, 3, 2]) == 13
    for w in range(1, 25):
        assert sub2ind([2, 4, 3], ind2sub([2, 4, 3], w)) == w
    with pytest.raises(TenkitError, match="worker id out of range"):
        ind2sub([2, 2], 5)
    g = GridPlan.even((9, 8, 7), (2, 1, 3))
    assert g.world == 6 and g.splits == [[5, 4], [8], [3, 2, 2]] and g.offsets[2] == [0, 3, 5]
    assert g.block(0) == ([0, 0, 0], [5, 8, 3]) and g.block(1) == ([5, 0, 0], [4, 8, 3])
    assert g.block(5) == ([5, 0, 5], [4, 8, 2])
    y = np.arange(9 * 8 * 7, dtype=np.float64).reshape((9, 8, 7), order="F")
    cover = np.zeros_like(y)
    for r in range(g.world):
        lo, ln = g.block(r)
        cover[lo[0]:lo[0] + ln[0], lo[1]:lo[1] + ln[1], lo[2]:lo[2] + ln[2]] += 1
        blk = g.local(y, r)
        assert blk.flags.f_contiguous and blk.shape == tuple(ln)
    assert (cover == 1).all()
    with pytest.raises(TenkitError, match="split lengths must sum to the mode dimension"):
        GridPlan((4, 4), [[2, 1], [4]])
    with pytest.raises(TenkitError, match="one split list per mode required"):
        GridPlan((4, 4), [[4]])
    assert default_grid(3, 8) == [2, 2, 2] and default_grid(3, 4) == [1, 1, 4] and default_grid(4, 2) == [1, 1, 1, 2]


def _block_worker(rank, world, port, grid_shape, q):
    """Block-grid sharding identity on the oracle: partial sketches of every mode (own rows of
    Z for a partitioned mode, zero elsewhere) and partial cores, summed through DistComm,
    equal the single-node products; the tk_comm struct carries the block."""
    try:
        import torch
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import pyoracle as O
        from paper_1412_1885_b200.dist import DistComm, GridPlan, exchange_capacity
        O.set_threads(1)
        dims, ranks, p = (13, 12, 11), (3, 3, 3), 2
        seed = (5, 0)
        y = O.add_noise(O.gen_tucker(dims, ranks, seed), 10.0, O.seed_derived(*seed, 0xAD0))
        plan = GridPlan.even(dims, grid_shape)
        lo, ln = plan.block(rank)
        yl = plan.local(y, rank)
        rts = [min(r + p, i) for r, i in zip(ranks, dims)]
        us = [O.gaussian_matrix(i, r, (9, n)) for n, (i, r) in enumerate(zip(dims, rts))]
        ul = [u[a:a + b] for u, a, b in zip(us, lo, ln)]
        comm = DistComm(lo[-1], dims[-1], exchange_capacity(dims, ranks, p), block_lo=lo, global_dims=dims)
        errs = []
        for n in range(3):
            om = O.gaussian_matrix(int(np.prod([rts[k] for k in range(3) if k != n])), rts[n], (11, n))
            full = O.unfold_times(O.ttm_all(y, us, n, True), n, om)
            part = O.unfold_times(O.ttm_all(yl, ul, n, True), n, om)
            zp = np.zeros_like(full)
            zp[lo[n]:lo[n] + ln[n]] = part
            comm.xbuf[: zp.size] = torch.from_numpy(zp.ravel(order="F"))
            assert comm.allreduce(zp.size) == 0
            got = comm.xbuf[: zp.size].numpy().reshape(full.shape, order="F")
            errs.append(float(np.abs(got - full).max() / np.abs(full).max()))
        g_full = O.ttm_all(y, us, -1, True)
        g_part = O.ttm_all(yl, ul, -1, True)
        comm.xbuf[: g_part.size] = torch.from_numpy(g_part.ravel(order="F"))
        comm.allreduce(g_part.size)
        g_got = comm.xbuf[: g_part.size].numpy().reshape(g_full.shape, order="F")
        errs.append(float(np.abs(g_got - g_full).max() / np.abs(g_full).max()))
        st = comm.as_struct()
        assert st.blocked == 1 and list(st.block_lo[:3]) == lo and list(st.global_dims[:3]) == list(dims)
        q.put((rank, errs, comm.calls))
        dist.destroy_process_group()
    except Exception as e:
        import traceback
        q.put((rank, repr(e) + traceback.format_exc(), -1))


def test_gloo_world4_block_grid_partials_reduce_to_single_node():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    grid = (2, 1, 2)
    procs = [ctx.Process(target=_block_worker, args=(r, 4, port, grid, q)) for r in range(4)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for rank, errs, calls in res:
        assert calls == 4, errs
        assert max(errs) < 1e-12, errs


# ---------------------------------------------------------------- MessageLog (dist.hpp:277-320)
def test_message_log_records_counts_and_ndjson():
    """MessageLog mirrors the reference's audit log: monotone seq, count(kind[, mode]), one
    JSON object per line (test_dist.cpp:186-201, 270-285)."""
    import io
    import json
    from paper_1412_1885_b200.dist import MessageLog, exchange_plan
    log = MessageLog()
    plan = exchange_plan("2i", (40, 36, 30), (5, 5, 5), 4)
    assert [p[2] for p in plan] == [0, 1, 2, 0, 1, 2, -1]
    for kind, tag, mode, rows in plan:
        log.append(kind, 1, -1, mode, tag, rows or 729, 9 if rows else 1)
    assert log.count("partial_product") == 6 and log.count("core_block") == 1
    assert log.count("partial_product", 1) == 2
    recs = log.records()
    assert all(b.seq > a.seq for a, b in zip(recs, recs[1:]))
    f = io.StringIO()
    log.write_ndjson(f)
    lines = f.getvalue().splitlines()
    assert len(lines) == len(recs)
    d = json.loads(lines[0])
    assert d == {"seq": 0, "kind": "partial_product", "source": 1, "dest": -1, "mode": 0, "tag": "z", "rows": 40,
                 "cols": 9}
    with pytest.raises(ValueError):
        log.append("bogus", 1, -1, 0, "z", 1, 1)
    assert [p[2] for p in exchange_plan("alg2", (8, 8, 8, 8), (2, 2, 2, 2), 1)] == [0, 1, 2, 3, -1]


def _log_worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1412_1885_b200.dist import DistComm, MessageLog, exchange_plan
        dims, ranks, p = (12, 10, 8), (3, 3, 3), 2
        comm = DistComm(0, dims[-1], 256, device="cpu")
        comm.log, comm.plan = MessageLog(), exchange_plan("alg2", dims, ranks, p)
        for n in range(3):  # the call sequence of one Alg. 2 decomposition: Z_0..Z_2, core
            comm.xbuf[: dims[n] * 5] = float(rank + 1)
            comm.allreduce(dims[n] * 5)
            assert float(comm.xbuf[0]) == 3.0
        comm.allreduce(125)
        q.put((rank, [tuple(r) for r in comm.log.records()]))
        dist.destroy_process_group()
    except Exception as e:
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))


def test_gloo_world2_exchanges_are_logged():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_log_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    for rank in (0, 1):
        recs = res[rank]
        assert isinstance(recs, list), recs
        assert [(r[1], r[2], r[4], r[5], r[6], r[7]) for r in recs] == [
            ("partial_product", rank + 1, 0, "z", 12, 5), ("partial_product", rank + 1, 1, "z", 10, 5),
            ("partial_product", rank + 1, 2, "z", 8, 5), ("core_block", rank + 1, -1, "core", 125, 1)]
