"""Pins the CPU oracle against the reference's own tensor/RNG tests.

Mirrors /root/reference/proj/tests/test_tensor.cpp and test_random.cpp (literal KATs and
properties), plus an independent numpy restatement of the counter RNG (random.hpp:12-71)."""
import numpy as np
import pytest

from helpers import np_key, np_mix64, np_normal, np_counter_unit, oracle_unfold, np_unfold


def rt(O, shape, seed):  # test_support.hpp:40-42 random_tensor
    flat = O.gaussian_matrix(int(np.prod(shape)), 1, (seed, 0)).ravel(order="F")
    return flat.reshape(shape, order="F")


def test_unfold_worked_2x2x2(O):  # test_tensor.cpp:10-22
    t = np.arange(1, 9, dtype=float).reshape((2, 2, 2), order="F")
    assert np.array_equal(O.unfold(t, 0), [[1, 3, 5, 7], [2, 4, 6, 8]])
    assert np.array_equal(O.unfold(t, 1), [[1, 2, 5, 6], [3, 4, 7, 8]])


def test_unfold_order1(O):  # test_tensor.cpp:24-30
    m = O.unfold(np.array([4.0, 5.0, 6.0]), 0)
    assert m.shape == (3, 1) and m[1, 0] == 5.0


@pytest.mark.parametrize("shape", [(4,), (3, 5), (3, 4, 2), (2, 3, 2, 4), (2, 2, 3, 2, 2)])
def test_unfold_matches_index_map(O, shape):  # test_tensor.cpp:32-40
    t = rt(O, shape, 100 + len(shape))
    for n in range(len(shape)):
        assert np.array_equal(O.unfold(t, n), oracle_unfold(t, n))
        assert np.array_equal(O.unfold(t, n), np_unfold(t, n))


def test_ttm_identity_and_unfold_product(O):  # test_tensor.cpp:61-76
    t = rt(O, (3, 4, 2), 7)
    for n in range(3):
        r = O.ttm(t, np.eye(t.shape[n]), n)
        assert np.array_equal(O.unfold(r, 0), O.unfold(t, 0))
    t = rt(O, (3, 4, 2), 8)
    for n in range(3):
        m = O.gaussian_matrix(5, t.shape[n], (9, n))
        r = O.ttm(t, m, n)
        ref = m @ O.unfold(t, n)
        assert np.linalg.norm(O.unfold(r, n) - ref) / np.linalg.norm(ref) < 1e-12


def test_ttm_ones_kat(O):  # test_tensor.cpp:78-85
    r = O.ttm(np.ones((2, 2)), np.ones((1, 2)), 0)
    assert r.shape == (1, 2) and r[0, 0] == 2.0 and r[0, 1] == 2.0


def test_unfold_times(O):  # test_tensor.cpp:87-95
    t = rt(O, (4, 3, 5), 11)
    for n in range(3):
        b = O.gaussian_matrix(t.size // t.shape[n], 6, (12, n))
        ref = O.unfold(t, n) @ b
        assert np.linalg.norm(O.unfold_times(t, n, b) - ref) / np.linalg.norm(ref) < 1e-13


def test_ttm_all_ascending_transposed(O):  # tensor.hpp:181-192
    t = rt(O, (5, 4, 3), 13)
    us = [O.gaussian_matrix(s, 2, (14, k)) for k, s in enumerate(t.shape)]
    for skip in (-1, 0, 1, 2):
        x = O.ttm_all(t, us, skip, True)
        ref = t
        for n in range(3):
            if n != skip:
                ref = np.moveaxis(np.tensordot(us[n].T, ref, axes=([1], [n])), 0, n)
        assert np.allclose(x, ref, rtol=1e-12, atol=1e-12)


def test_fit_kats(O):  # test_tensor.cpp:168-180
    y = rt(O, (3, 3), 18)
    assert O.fit(y, y) == pytest.approx(1.0)
    assert O.fit(y, np.zeros((3, 3))) == pytest.approx(0.0)
    assert O.fit(np.array([3.0, 4.0]), np.array([3.0, 0.0])) == pytest.approx(0.2)
    with pytest.raises(ValueError, match="zero norm"):
        O.fit(np.zeros((3, 3)), y)


def test_shape_invariants(O):  # test_tensor.cpp:182-187
    with pytest.raises(ValueError):
        O.unfold(np.zeros((2, 2)), 2)


# ------------------------------------------------------------------ random.hpp
def test_gaussian_deterministic_and_streams(O):  # test_random.cpp:10-21
    a = O.gaussian_matrix(20, 5, (42, 7))
    assert np.array_equal(a, O.gaussian_matrix(20, 5, (42, 7)))
    assert np.abs(O.gaussian_matrix(8, 3, (42, 0)) - O.gaussian_matrix(8, 3, (42, 1))).max() > 0


def test_gaussian_moments(O):  # test_random.cpp:23-30
    m = O.gaussian_matrix(10000, 10, (123, 0))
    assert abs(m.mean()) < 0.05
    v = m.var(ddof=1)
    assert 0.9 < v < 1.1


def test_sub_block_reproducible(O):  # test_random.cpp:32-39
    full = O.gaussian_matrix(40, 6, (99, 3))
    rows = [0, 3, 5, 17, 18, 39]
    assert np.array_equal(O.gaussian_rows(40, 6, (99, 3), rows), full[rows])


def test_normal_at_matches_layout(O):  # test_random.cpp:41-47
    m = O.gaussian_matrix(7, 4, (5, 11))
    for j in range(4):
        for i in range(7):
            assert O.normal_at(5, 11, j * 7 + i) == m[i, j]


def test_derived_streams(O):  # test_random.cpp:49-54
    base = (1, 2)
    assert O.seed_derived(*base, 10) == O.seed_derived(*base, 10)
    assert O.seed_derived(*base, 10) != O.seed_derived(*base, 11)
    assert O.seed_derived(*base, 10, 4) != O.seed_derived(*base, 10, 5)


def test_exponential_mean(O):  # test_random.cpp:56-62 (exponential_at = -mean*log(unit))
    u = np.array([O.uniform_at(77, 0, i) for i in range(40000)])
    assert (-10.0 * np.log(u)).mean() == pytest.approx(10.0, abs=0.25)


def test_rng_bit_exact_vs_numpy_restatement(O):
    """Independent numpy restatement of random.hpp:12-71 agrees bit-for-bit (u64 keys)
    and to <=1 ulp on the Box-Muller normals (libm vs numpy transcendental kernels)."""
    for x in [0, 1, 2**63, 0xDEADBEEF, 2**64 - 1]:
        assert O.mix64(x) == int(np_mix64(np.uint64(x)))
    for root, stream in [(0, 0), (33, 0), (7, 123456789)]:
        key = O.seed_key(root, stream)
        assert key == int(np_key(root, stream))
        idx = np.arange(0, 2000, dtype=np.uint64)
        u = np_counter_unit(key, idx)
        assert all(u[i] == O.uniform_at(root, stream, int(i)) for i in range(0, 2000, 97))
        ref = O.gaussian_matrix(2000, 1, (root, stream)).ravel()
        assert np.max(np.abs(np_normal(key, idx) - ref) / np.maximum(np.abs(ref), 1e-300)) < 4e-16


def test_threaded_gaussian_fill_is_split_invariant(O):
    """The oracle splits large gaussian fills over host threads at even (Box-Muller pair)
    boundaries: every entry stays normal_at(seed, index) (random.hpp:63-71, 124-138)."""
    O.set_threads(1)
    a = O.gaussian_matrix(3_000_001, 1, (3, 4))
    O.set_threads(7)
    b = O.gaussian_matrix(3_000_001, 1, (3, 4))
    O.set_threads(1)
    assert np.array_equal(a, b)
    assert a[2_999_999, 0] == O.normal_at(3, 4, 2_999_999) and a[3_000_000, 0] == O.normal_at(3, 4, 3_000_000)
