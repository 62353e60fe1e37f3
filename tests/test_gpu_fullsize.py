"""BASELINE configs 3 and 4 at their FULL sizes (2400^3 fp32 = 55 GB, 300^4 fp32 = 32 GB) and cfg 5's
per-GPU slab at 4 GPUs (4000 x 4000 x 1000 fp32 = 64 GB, ranks 50, r~ 60) on one B200:

* oracle parity (north star: U_n, core and fit at 1e-3 in fp32; 1e-5 for the fp64 mode,
  precision='fp64': fp64 arithmetic over the same fp32 values): the CPU oracle's streamed-slab
  rand_tucker_2i (oracle/tenkit_oracle.cpp rand_tucker_2i_streamed: the reference's control flow,
  tucker.hpp:136-169, with every ttm_all accumulated over last-mode slabs as dist.hpp:496-596
  streams blocks; fp64 on the same fp32 values) against the device model: the subspace of ALL
  r~ columns of every factor, the core after aligning bases, and the fit;
* determinism: two decompositions of the same Y are bit-identical (tucker.hpp's contract,
  test_tucker.cpp:114-121), the second one a CUDA-graph replay;
* orthonormal factors (<= 1e-10, test_tucker.cpp:105-112) and the sign rule (tucker.hpp:39-45);
* the Gram identity ||Y||^2 - ||G||^2 = ||Y - G x U||^2 against the streamed fit kernel;
* the generator's true factors lie in the computed subspaces (signal captured at 20/30 dB);
* shared Y passes == one pass per step (the reference's structure) to the fp32 bar.

Data: the bench's seeded generators on the device (bench.hpp:46-112 seeds, chunked into fp32).
The oracle's pivot / sign margins of every range step are logged (TENKIT_PARITY_LOG=path.jsonl)."""
import json
import os
import time

import numpy as np
import pytest

from helpers import orthonormality_defect, subspace_dist

pytestmark = pytest.mark.gpu

F32_TOL = 1e-3  # north_star: fp32 configs agree with the fp64 oracle within 1e-3
# relative margin of a discrete decision (ColPiv pivot, sign rule) that fp32-accurate
# contractions resolve; below it the fp32 path may take the other branch
RESOLVABLE = 1e-5


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1412_1885_b200 as P
    return P


def _true_factors(cfg):
    from paper_1412_1885_b200.generators import bench_seeds, gaussian_flat, gen_factor_seed, uniform_matrix
    data_seed, _ = bench_seeds(cfg.get("seed", 0))
    out = []
    for n, i in enumerate(cfg["dims"]):
        if cfg["gen"] == "tucker":
            r = int(cfg["mlrank"][n])
            a = gaussian_flat(int(i) * r, gen_factor_seed(data_seed, n)).view(r, int(i)).t().cpu().numpy()
        else:
            a = uniform_matrix(int(i), int(cfg["cp_rank"]), gen_factor_seed(data_seed, n))
        out.append(np.asarray(a, dtype=np.float64))
    return out


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def _gram_fit(ysq, core):
    return 1.0 - float(np.sqrt(max(0.0, 1.0 - float(np.sum(np.square(core))) / ysq)))


def _log(rec):
    path = os.environ.get("TENKIT_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    print(json.dumps(rec))


@pytest.mark.parametrize("name,capture_tol", [("cfg3", 0.05), ("cfg4", 0.05), ("cfg5slab", 0.05)])
def test_full_size_config(P, O, name, capture_tol):
    import torch
    import bench
    from paper_1412_1885_b200.generators import bench_seeds, generate_as
    cfg = dict(bench.CONFIGS[name], seed=0)
    dims = [int(d) for d in cfg["dims"]]
    y = generate_as(cfg, torch.float32)
    yd = P.DenseTensor(dims, y)
    _, alg = bench_seeds(0)
    ranks, p = list(cfg["ranks"]), int(cfg["p"])
    runs = [P.rand_tucker_2i(yd, ranks, p, alg, sync_ranks=False, out="device") for _ in range(3)]
    a, b = runs[1].to_host(), runs[2].to_host()  # runs[2] replays the graph captured by runs[1]
    if os.environ.get("TENKIT_TTM_PATH", "0") != "1":  # (the FFMA-only A/B path cannot lead a pass with mode 0)
        assert a.stats["passes"] == 3  # r~ = 60 too: the K-major tcgen05 pass leads over mode 0
    np.testing.assert_array_equal(a.core, b.core)
    for u, v in zip(a.factors, b.factors):
        np.testing.assert_array_equal(u, v)

    truth = _true_factors(cfg)
    for u, t in zip(a.factors, truth):
        assert u.shape[1] == min(ranks[0] + p, u.shape[0])
        assert orthonormality_defect(u) < 1e-10
        imax = np.argmax(np.abs(u), axis=0)  # sign rule: the largest-|.| entry of each column is positive
        assert np.all(u[imax, np.arange(u.shape[1])] > 0)
        resid = t - u @ (u.T @ t)
        miss = np.linalg.norm(resid) / np.linalg.norm(t)
        assert miss < capture_tol, f"true factor outside the computed subspace: {miss:.3e}"

    # Gram identity vs the streamed ||Y - Yhat|| (fp64 sums over the fp32 Y)
    fit, rnorm, ynorm = P.model_fit(yd, runs[1], norms=True)
    gsq = float(np.sum(a.core ** 2))
    assert abs((ynorm ** 2 - gsq) - rnorm ** 2) <= 1e-4 * ynorm ** 2
    assert fit > (0.85 if cfg["snr"] <= 20 else 0.95)

    # shared Y passes vs the reference's one pass per step (fp32 bar, all r~ columns; asserted
    # below unless a discrete decision of the reference is closer than fp32 can resolve)
    s = P.rand_tucker_2i(yd, ranks, p, alg, sync_ranks=False, out="device", one_pass_per_step=True)
    assert s.stats["passes"] == 2 * len(dims)
    sh = s.to_host()
    d_steps = [subspace_dist(u, v) for u, v in zip(a.factors, sh.factors)]
    assert abs(P.model_fit(yd, s) - fit) < 1e-4

    # the fp64 mode (tk_tucker_opts.precision = 1): fp64 arithmetic over the same fp32 values
    t0 = time.perf_counter()
    prec = P.rand_tucker_2i(yd, ranks, p, alg, sync_ranks=False, out="host", precision="fp64")
    t_prec = time.perf_counter() - t0

    # ---- the oracle on the same fp32 bytes (host copy; the device tensor is freed first)
    yh = y.cpu().numpy()
    del y, yd, runs, s
    torch.cuda.empty_cache()
    O.set_threads(os.cpu_count() or 1)
    t0 = time.perf_counter()
    g_ref, u_ref, margins = O.rand_tucker_2i_streamed(yh, dims, ranks, p, (alg.root, alg.stream))
    t_oracle = time.perf_counter() - t0
    O.set_threads(1)
    ysq = 0.0
    for c0 in range(0, yh.size, 1 << 27):
        c = yh[c0:c0 + (1 << 27)].astype(np.float64)
        ysq += float(np.dot(c, c))
    del yh
    sub = [subspace_dist(u, v) for u, v in zip(a.factors, u_ref)]
    aligned = O.ttm_all(a.core, [u.T @ v for u, v in zip(a.factors, u_ref)], -1, False)
    core_err = _rel(aligned, g_ref)
    f_got, f_ref = _gram_fit(ysq, a.core), _gram_fit(ysq, g_ref)
    sub64 = [subspace_dist(u, v) for u, v in zip(prec.factors, u_ref)]
    core64 = _rel(O.ttm_all(prec.core, [u.T @ v for u, v in zip(prec.factors, u_ref)], -1, False), g_ref)
    _log({"test": "full_size_oracle", "config": name, "subspace_all_cols": sub, "core_rel": core_err,
          "fit": f_got, "fit_oracle": f_ref, "shared_vs_per_step": d_steps,
          "fp64_mode_subspace": sub64, "fp64_mode_core_rel": core64, "fp64_mode_s": round(t_prec, 2),
          "pivot_margin_min": float(margins[:, 0].min()), "sign_margin_min": float(margins[:, 1].min()),
          "margins": margins.tolist(), "oracle_s": round(t_oracle, 1), "threads": os.cpu_count()})
    for u, v in zip(a.factors, u_ref):
        assert u.shape == v.shape
    # the fp64 mode reproduces the reference's decisions and values at the fp64 bar (1e-5)
    assert max(sub64) < 1e-5 and core64 < 1e-5, (sub64, core64)
    # the device reports the same decision margins as the oracle (its own fp32 values)
    dev_pm, dev_sm = np.array(a.stats["pivot_margin"]), np.array(a.stats["sign_margin"])
    assert np.all(np.abs(dev_pm - margins[:, 0]) < 1e-3 + 0.1 * margins[:, 0])
    assert np.all(np.abs(dev_sm - margins[:, 1]) < 1e-3 + 0.1 * margins[:, 1])
    assert abs(f_got - f_ref) < F32_TOL, (f_got, f_ref)
    if float(margins.min()) >= RESOLVABLE:
        assert max(sub) < F32_TOL, sub
        assert core_err < F32_TOL, core_err
        assert max(d_steps) < F32_TOL, d_steps
    else:
        # a reference decision (pivot / sign rule) within fp32 resolution: flagged by the device
        assert min(float(dev_pm.min()), float(dev_sm.min())) < 10 * RESOLVABLE
