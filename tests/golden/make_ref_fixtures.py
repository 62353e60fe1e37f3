"""Reference-RUN fixtures: outputs of the reference's own hot-path code.

oracle/_ref/libtenkit_ref.so is /root/reference/proj/include/tenkit/{tensor,random,
range_finder,tucker}.hpp compiled unmodified from where they lie against oracle/ref_shim
(an eager Eigen-API stand-in: products as fixed-order loops, ColPivHouseholderQR ->
LAPACK dgeqp3, SelfAdjointEigenSolver -> dsyev). Every input below is built with the
reference's own functions (gaussian_matrix, ttm), every output is the reference's
rand_tucker_2i / rand_tucker / ttm / unfold_times / orthonormal_basis (+ fix_column_signs).
Only this script runs the reference (it needs /root/reference); the committed
ref_fixtures.npz is what tests/test_ref_fixtures.py (oracle, CPU) and
tests/test_gpu_ref_fixtures.py (device) check against. Run:
    python tests/golden/make_ref_fixtures.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle as O  # noqa: E402

# (name, dims, tucker ranks of the data, noise rel. amplitude, decomposition ranks, oversample)
CASES = [
    ("t3", (24, 20, 18), (4, 4, 4), 0.1, (4, 4, 4), 3),
    ("t3b", (30, 26, 22), (5, 3, 4), 0.3, (5, 4, 4), 4),
    ("t4", (10, 9, 8, 7), (3, 3, 3, 3), 0.1, (3, 3, 3, 3), 2),
    ("t2", (40, 33), (5, 5), 0.05, (5, 5), 3),
    ("wide", (12, 50, 45), (6, 6, 6), 0.1, (10, 6, 6), 4),
    ("rankdrop", (16, 14, 12), (2, 2, 2), 0.0, (4, 4, 4), 2),
]


def ref_tucker_data(dims, mlr, noise, seed):
    """Y = core x_0 A_0 ... + noise, every draw the reference's gaussian_matrix (random.hpp:85-100)
    and every contraction the reference's ttm (tensor.hpp:151-176)."""
    core = O.ref_gaussian_matrix(int(np.prod(mlr)), 1, (seed, 1)).reshape(mlr, order="F")
    y = core
    for n, (i, r) in enumerate(zip(dims, mlr)):
        y = O.ref_ttm(y, O.ref_gaussian_matrix(i, r, (seed, 10 + n)), n)
    if noise > 0:
        e = O.ref_gaussian_matrix(int(np.prod(dims)), 1, (seed, 99)).reshape(dims, order="F")
        y = y + noise * np.linalg.norm(y) / np.linalg.norm(e) * e
    return y


def main():
    O.ref_lib()
    out = {}
    # counter RNG (random.hpp:12-100): normals and derived streams
    seeds = [(0, 0), (33, 0), (7, 123456789), (2**63 + 5, 17)]
    out["rng_seeds"] = np.array(seeds, dtype=np.uint64)
    out["rng_normals"] = np.stack([O.ref_gaussian_matrix(9, 3, s).ravel(order="F") for s in seeds])
    out["rng_derived"] = np.array([O.ref_lib().tkr_seed_derived(33, 0, t) for t in (0x0A2, 0x0A3, 0x0B3, 0x0B4, 0xC0DE)],
                                  dtype=np.uint64)
    # ttm / unfold_times (tensor.hpp:151-209)
    t = O.ref_gaussian_matrix(7 * 6 * 5, 1, (3, 4)).reshape((7, 6, 5), order="F")
    out["k_t"] = t
    for n in range(3):
        m = O.ref_gaussian_matrix(4, t.shape[n], (5, n))
        out[f"k_ttm_m{n}"] = m
        out[f"k_ttm_out{n}"] = O.ref_ttm(t, m, n)
        b = O.ref_gaussian_matrix(t.size // t.shape[n], 3, (6, n))
        out[f"k_ut_b{n}"] = b
        out[f"k_ut_out{n}"] = O.ref_unfold_times(t, n, b)
    # orthonormal_basis + fix_column_signs (range_finder.hpp:18-29, tucker.hpp:39-45), incl. rank drop
    z = O.ref_gaussian_matrix(40, 7, (11, 3))
    z[:, 2] = 2.0 * z[:, 0] - z[:, 5]
    out["qr_z"], out["qr_u"] = z, O.ref_orthonormal_basis(z)
    z2 = O.ref_gaussian_matrix(300, 12, (12, 3)) @ np.diag(np.linspace(1.0, 3.0, 12))
    out["qr_z2"], out["qr_u2"] = z2, O.ref_orthonormal_basis(z2)
    # the decompositions (tucker.hpp:108-169), fp64 data and the same data rounded to fp32
    names = []
    for name, dims, mlr, noise, ranks, p in CASES:
        y = ref_tucker_data(dims, mlr, noise, 101 + len(names))
        for tag, yy in (("f64", y), ("f32", y.astype(np.float32).astype(np.float64))):
            key = f"{name}_{tag}"
            out[f"{key}_y"] = yy
            g, us = O.ref_rand_tucker_2i(yy, ranks, p, (1, 2))
            out[f"{key}_2i_core"] = g
            for n, u in enumerate(us):
                out[f"{key}_2i_u{n}"] = u
            g, us = O.ref_rand_tucker(yy, ranks, p, (3, 4))
            out[f"{key}_a2_core"] = g
            for n, u in enumerate(us):
                out[f"{key}_a2_u{n}"] = u
        out[f"{name}_ranks"] = np.array(ranks)
        out[f"{name}_p"] = np.array(p)
        names.append(name)
    out["cases"] = np.array(names)
    path = os.path.join(HERE, "ref_fixtures.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
