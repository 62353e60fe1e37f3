"""Shared test helpers: independent numpy restatements used to cross-check the oracle."""
import numpy as np

MASK = np.uint64(0xFFFFFFFFFFFFFFFF)


def np_mix64(x):
    """splitmix64 finalizer (random.hpp:12-18) in numpy uint64 (wrapping) arithmetic."""
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def np_hash_combine(a, b):
    with np.errstate(over="ignore"):
        a = np.uint64(a)
        return np_mix64(a ^ (np_mix64(np.uint64(b)) + np.uint64(0x9E3779B97F4A7C15) + (a << np.uint64(6)) + (a >> np.uint64(2))))


def np_key(root, stream):
    return np_hash_combine(np_mix64(np.uint64(root)), np.uint64(stream))


def np_counter_unit(key, idx):
    with np.errstate(over="ignore"):
        bits = np_mix64(np.uint64(key) + np.asarray(idx, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15))
    return ((bits >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0**-53


def np_normal(key, idx):
    idx = np.asarray(idx, dtype=np.uint64)
    pair = idx >> np.uint64(1)
    u1 = np_counter_unit(key, np.uint64(2) * pair)
    u2 = np_counter_unit(key, np.uint64(2) * pair + np.uint64(1))
    r = np.sqrt(-2.0 * np.log(u1))
    ang = 6.283185307179586476925287 * u2
    return np.where((idx & np.uint64(1)) == 1, r * np.sin(ang), r * np.cos(ang))


def oracle_unfold(t, mode):
    """Element-wise index-map unfold (test_support.hpp:15-38), independent of the oracle."""
    shape = t.shape
    cols = int(np.prod([s for k, s in enumerate(shape) if k != mode]))
    out = np.zeros((shape[mode], cols))
    for sub in np.ndindex(*shape):
        col, stride = 0, 1
        for k, s in enumerate(shape):
            if k == mode:
                continue
            col += sub[k] * stride
            stride *= s
        out[sub[mode], col] = t[sub]
    return out


def np_unfold(t, mode):
    return np.reshape(np.moveaxis(t, mode, 0), (t.shape[mode], -1), order="F")


def subspace_dist(u, v):
    """||U U^T - V V^T||_F (the north-star parity metric)."""
    return float(np.linalg.norm(u @ u.T - v @ v.T))


def orthonormality_defect(u):
    return float(np.abs(u.T @ u - np.eye(u.shape[1])).max()) if u.shape[1] else 0.0


def max_principal_angle(qa, qb):
    resid = qb - qa @ (qa.T @ qb)
    s = np.linalg.svd(resid, compute_uv=False)
    return float(np.arcsin(min(1.0, s[0] if s.size else 0.0)))


def transpositions_to_perm(t):
    p = list(range(len(t)))
    for k, j in enumerate(t):
        p[k], p[j] = p[j], p[k]
    return p
