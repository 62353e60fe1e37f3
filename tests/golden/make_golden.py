"""Regenerates the golden fixtures in this directory from the CPU oracle (oracle/).

The reference (tenkit) cannot be built in this image (no Eigen3 / Catch2), and its own
suite holds no golden vectors for the sketch / QR / core, so these fixtures
are the oracle's outputs on seeded inputs defined entirely by the reference's counter RNG
and generators. They pin the oracle against regressions and give the device tests a
fixed target. Run:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as O  # noqa: E402


def main():
    O.build()
    O.set_threads(1, use_blas=False)  # fixed-order loops: reproducible bit patterns
    out = {}
    # counter RNG (random.hpp:12-100)
    seeds = [(0, 0), (33, 0), (7, 123456789)]
    out["rng_seeds"] = np.array(seeds, dtype=np.uint64)
    out["rng_keys"] = np.array([O.seed_key(*s) for s in seeds], dtype=np.uint64)
    out["rng_normals"] = np.stack([O.gaussian_matrix(16, 1, s).ravel() for s in seeds])
    out["rng_uniforms"] = np.array([[O.uniform_at(*s, i) for i in range(16)] for s in seeds])
    out["rng_derived"] = np.array([O.seed_derived(33, 0, 0x0A3, n)[1] for n in range(4)], dtype=np.uint64)
    # pivoted QR (range_finder.hpp:18-29) + sign rule (tucker.hpp:39-45)
    z = O.gaussian_matrix(40, 7, (11, 3))
    z[:, 2] = 2.0 * z[:, 0] - z[:, 5]  # rank 6
    u, d = O.orthonormal_basis(z, diagnostics=True)
    out["qr_z"], out["qr_u"] = z, O.fix_column_signs(u)
    out["qr_perm"], out["qr_rdiag"] = d["perm"], d["rdiag"]
    # rand_tucker_2i / rand_tucker on a seeded noisy Tucker tensor (bench.hpp generators)
    data = O.seed_derived(0, 0, 0xDA7A, 0)
    y = O.add_noise(O.gen_tucker((20, 18, 16), (4, 4, 4), data), 10.0, O.seed_derived(*data, 0xAD0))
    out["tucker_y"] = y
    g, us = O.rand_tucker_2i(y, (4, 4, 4), 3, (7, 0))
    out["rt2i_core"] = g
    for n, uu in enumerate(us):
        out[f"rt2i_u{n}"] = uu
    g1, us1 = O.rand_tucker(y, (4, 4, 4), 3, (7, 0))
    out["rt_core"] = g1
    for n, uu in enumerate(us1):
        out[f"rt_u{n}"] = uu
    a, trace, its = O.ffcp(g, us, 3, O.NONE, 0.0, 50, 1e-9, (8, 0))
    out["ffcp_trace"] = trace
    for n, aa in enumerate(a):
        out[f"ffcp_a{n}"] = aa
    np.savez_compressed(os.path.join(HERE, "oracle_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "oracle_golden.npz"), sorted(out))


if __name__ == "__main__":
    main()
