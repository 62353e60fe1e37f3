"""The benchmark workload itself: device generator parity (bench.hpp:46-112 restated on the
device) and parity of the decomposition on BASELINE configs[1]'s shape, at a reduced size
against the oracle and at full size (1000^3 fp32) through size-independent properties
plus the oracle on the same Y (fp64, all host cores)."""
import os

import numpy as np
import pytest

from helpers import orthonormality_defect, subspace_dist

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1412_1885_b200 as P
    return P


def test_device_generators_match_oracle(P, O):
    from paper_1412_1885_b200 import generators as G
    data, _ = G.bench_seeds(0)
    y = G.gen_tucker_device((30, 26, 22), (4, 3, 2), data).cpu().numpy().reshape((30, 26, 22), order="F")
    ref = O.gen_tucker((30, 26, 22), (4, 3, 2), (data.root, data.stream))
    assert np.abs(y - ref).max() < 1e-12 * np.abs(ref).max()
    yn = G.add_noise_device(G.gen_tucker_device((30, 26, 22), (4, 3, 2), data), 20.0, data.derived(0xAD0))
    refn = O.add_noise(ref, 20.0, O.seed_derived(data.root, data.stream, 0xAD0))
    assert np.abs(yn.cpu().numpy().reshape(ref.shape, order="F") - refn).max() < 1e-12 * np.abs(refn).max()
    yc = G.gen_cp_device((12, 10, 8, 6), 3, data, uniform=True).cpu().numpy().reshape((12, 10, 8, 6), order="F")
    refc, _ = O.gen_cp((12, 10, 8, 6), 3, O.CP_UNIFORM, (data.root, data.stream))
    assert np.abs(yc - refc).max() < 1e-12 * np.abs(refc).max()
    yca = G.add_noise_device(G.gen_cp_device((12, 10, 8, 6), 3, data), 30.0, data.derived(0xAD0), abs_noise=True)
    refca = O.add_noise(refc, 30.0, O.seed_derived(data.root, data.stream, 0xAD0), abs_noise=True)
    assert np.abs(yca.cpu().numpy().reshape(refc.shape, order="F") - refca).max() < 1e-12 * np.abs(refca).max()


def _gram_fit(y64_flat, core):
    ysq = float(np.dot(y64_flat, y64_flat))
    return 1.0 - np.sqrt(max(0.0, 1.0 - float(np.sum(core ** 2)) / ysq))


def _check_against_oracle(P, O, dims, mlrank, ranks, p, threads=None):
    import torch
    from paper_1412_1885_b200 import generators as G
    cfg = dict(dims=dims, gen="tucker", mlrank=mlrank, snr=20.0)
    y64 = G.generate(cfg)
    y32 = y64.float()
    del y64
    _, alg = G.bench_seeds(0)
    m = P.rand_tucker_2i(P.DenseTensor(dims, y32), ranks, p, alg, sync_ranks=False, out="device").to_host()
    yh = y32.double().cpu().numpy()
    del y32
    torch.cuda.empty_cache()
    O.set_threads(threads or os.cpu_count() or 1)
    g_ref, u_ref = O.rand_tucker_2i(yh.reshape(dims, order="F"), ranks, p, (alg.root, alg.stream))
    O.set_threads(1)
    for u, v in zip(m.factors, u_ref):
        assert u.shape == v.shape
        assert orthonormality_defect(u) < 1e-10
        assert subspace_dist(u, v) < 1e-3
    f_got, f_ref = _gram_fit(yh, m.core), _gram_fit(yh, g_ref)
    assert abs(f_got - f_ref) < 1e-3
    assert f_got > 0.85  # 20 dB noise: the r~ = 30 Tucker model keeps ~90% fit
    return f_got


def test_config2_shape_reduced(P, O):
    _check_against_oracle(P, O, (240, 220, 200), (20, 20, 20), (20, 20, 20), 10)


def test_config2_full_size(P, O):
    """BASELINE configs[1] at full size: 1000^3 fp32 (4 GB), oracle on the same Y in fp64."""
    _check_against_oracle(P, O, (1000, 1000, 1000), (20, 20, 20), (20, 20, 20), 10)


@pytest.mark.parametrize("gen", ["tucker", "cp_uniform"])
def test_chunked_generation_matches_full(P, gen):
    """generate_as (chunked along the last mode, bounded fp64 temporaries; cfg 3/4 sizes)
    reproduces generate(); a full-sigma sample is the leading slab of the full tensor."""
    from paper_1412_1885_b200.generators import generate, generate_as
    import torch
    cfg = dict(dims=(20, 18, 33), gen=gen, mlrank=(3, 4, 2), cp_rank=3, snr=15.0, abs_noise=(gen != "tucker"))
    full = generate(cfg).cpu().numpy()
    got = generate_as(cfg, torch.float64, chunk_elems=20 * 18 * 5).cpu().numpy()
    np.testing.assert_allclose(got, full, rtol=0, atol=1e-12 * np.abs(full).max())
    part = generate_as(cfg, torch.float64, slab=(0, 7), full_sigma=True, chunk_elems=20 * 18 * 4).cpu().numpy()
    np.testing.assert_allclose(part, full[: 20 * 18 * 7], rtol=0, atol=1e-12 * np.abs(full).max())
    f32 = generate_as(cfg, torch.float32).cpu().numpy()
    np.testing.assert_array_equal(f32, full.astype(np.float32))
