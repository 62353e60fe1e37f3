"""The C++ host mirror (include/tenkit_b200.hpp) — the reference's own API surface
(DenseTensor / TuckerModel / rand_tucker_2i / ffcp, tucker.hpp:136-169, ffcp.hpp:94-194)
over the C-ABI — compiled with g++ as a reference caller would, no Python in the loop.
CPU: it builds and fails loudly (std::runtime_error) without a device.
GPU: its results equal the oracle's on the same seeded inputs."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEMO = os.path.join(ROOT, "examples", "_build", "cpp_mirror_demo")
ARGS = ["20", "18", "16", "3", "2", "3"]


@pytest.fixture(scope="module")
def demo():
    from paper_1412_1885_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("library not built")
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return DEMO


def parse(out):
    d = {"factor": [], "fit": []}
    for line in out.splitlines():
        k, *v = line.split()
        if k == "factor":
            d["factor"].append(tuple(int(x) for x in v))
        elif k == "fit":
            d["fit"].append(float(v[0]))
        elif k in ("core_sq", "y_sq"):
            d[k] = float(v[0])
        elif k in ("iterations", "gram_kept"):
            d[k] = int(v[0])
        elif k == "gram_defect":
            d[k] = float(v[0])
    return d


def test_cpp_mirror_fails_loudly_without_device(demo):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = subprocess.run([demo] + ARGS, capture_output=True, text=True)
    assert r.returncode == 4 and "runtime_error: tenkit:" in r.stdout


@pytest.mark.gpu
def test_cpp_mirror_matches_oracle(demo, O):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    r = subprocess.run([demo] + ARGS, capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    got = parse(r.stdout)
    fs = [O.gaussian_matrix(d, 3, O.seed_derived(0, 0, t)) for t, d in zip((1, 2, 3), (20, 18, 16))]
    core = O.gaussian_matrix(27, 1, O.seed_derived(0, 0, 4)).reshape((3, 3, 3), order="F")
    y = O.ttm_all(core, fs, -1, transpose=False)
    g, us = O.rand_tucker_2i(y, (3, 3, 3), 2, (7, 0))
    assert abs(got["y_sq"] - float(np.sum(y ** 2))) <= 1e-12 * float(np.sum(y ** 2))
    # exact-rank data: the rank-5 sketch captures Y, ||G||^2 = ||Y||^2 (fp64 tolerance 1e-5)
    assert abs(got["core_sq"] - float(np.sum(g ** 2))) <= 1e-5 * float(np.sum(y ** 2))
    assert got["factor"] == [(u.shape[0], u.shape[1]) for u in us]
    _, trace, its = O.ffcp(g, us, 3, O.NONE, 0.0, 30, 0.0, (8, 0))
    assert got["iterations"] == its
    np.testing.assert_allclose(got["fit"], trace, rtol=0, atol=1e-7)
    # gram_orthonormalize of a 15 + 25 row split (test_range_finder.cpp:66-77)
    assert got["gram_kept"] == 5 and got["gram_defect"] < 1e-10
