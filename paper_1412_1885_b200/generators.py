"""Seeded synthetic workloads of the reference benchmark (bench.hpp:46-112, 410-437) built on
the device: Tucker (Gaussian core + Gaussian factors) or CP (Gaussian / U(0,1) factors)
ground truth, plus realised-SNR Gaussian or |Gaussian| noise. Every random entry is the
reference's counter RNG at the reference's index (random.hpp:85-138), so the tensors are
the ones the reference's generators produce (up to fp64 rounding of the contractions).

The U(0,1) factors (configs 1, 4) and |N| noise (config 4) are the BASELINE configs'
additions, defined by mirroring bench.hpp:63-71: entry (i, j) of factor n is
uniform_at(gen_factor_seed(seed, n), j*I_n + i); noise is |gaussian_tensor(...)|.
"""
from __future__ import annotations

import numpy as np

from .tenkit import Context, SeedSpec, _ctx, _dptr, _lib

_GOLD = 0x9E3779B97F4A7C15


def _np_mix64(x):
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + np.uint64(_GOLD)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def uniform_matrix(rows: int, cols: int, seed: SeedSpec) -> np.ndarray:
    """uniform_at(seed, j*rows + i) in (0, 1] (random.hpp:48-56, 74-76), column-major."""
    idx = np.arange(rows * cols, dtype=np.uint64)
    with np.errstate(over="ignore"):
        bits = _np_mix64(np.uint64(seed.key()) + idx * np.uint64(_GOLD))
    v = ((bits >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0**-53
    return v.reshape((rows, cols), order="F")


def gaussian_flat(n: int, seed: SeedSpec, context: Context | None = None, offset: int = 0):
    """Flat fp64 CUDA tensor of gaussian_tensor / gaussian_matrix draws (random.hpp:85-138):
    entries offset .. offset + n - 1 of the seed's flat counter stream."""
    import torch
    ctx = _ctx(context)  # launches on torch's current stream: ordered with the torch ops below
    out = torch.empty(max(int(n), 1), dtype=torch.float64, device="cuda")
    if offset:
        _lib.check(ctx.lib.tk_gaussian_fill(ctx.handle, int(n), int(offset), seed.root, seed.stream, _dptr(out)))
    else:
        _lib.check(ctx.lib.tk_gaussian_matrix(ctx.handle, int(n), 1, seed.root, seed.stream, _dptr(out)))
    return out[: int(n)]


def gaussian_block(global_dims, lo, ln, seed: SeedSpec, context: Context | None = None):
    """Flat fp64 CUDA tensor (column-major block ln) of gaussian_tensor(global_dims, seed)
    restricted to the block starting at `lo`: every entry drawn at its global flat index
    (tk_gaussian_fill_block)."""
    import torch
    ctx = _ctx(context)
    n = int(np.prod([int(x) for x in ln]))
    out = torch.empty(max(n, 1), dtype=torch.float64, device="cuda")
    arr = lambda xs: (_lib.I64 * len(xs))(*[int(x) for x in xs])
    _lib.check(ctx.lib.tk_gaussian_fill_block(ctx.handle, len(global_dims), arr(global_dims), arr(lo), arr(ln),
                                              seed.root, seed.stream, _dptr(out)))
    return out[:n]


def gen_factor_seed(seed: SeedSpec, n: int) -> SeedSpec:  # bench.hpp:46-48
    return seed.derived(0x9E4, n)


def _colmajor_einsum(core, factors):
    """Y = core x_0 A_0 ... x_{N-1} A_{N-1} as a flat column-major fp64 CUDA tensor."""
    import torch
    order = len(factors)
    letters_r = "abcdefgh"[:order]
    letters_i = "ijklmnop"[:order]
    # row-major views with reversed mode order are the column-major layouts
    spec = letters_r[::-1] + "," + ",".join(letters_i[n] + letters_r[n] for n in range(order)) + "->" + letters_i[::-1]
    return torch.einsum(spec, core, *factors).contiguous().view(-1)


def _rows(a, n, order, last_rows, block):
    """Rows of factor n this block uses: block=(lo, ln) lists, or last_rows=(off, len) of the last mode."""
    if block is not None:
        return a[int(block[0][n]):int(block[0][n]) + int(block[1][n])]
    if last_rows is not None and n == order - 1:
        return a[int(last_rows[0]):int(last_rows[0]) + int(last_rows[1])]
    return a


def gen_tucker_device(dims, mlranks, seed: SeedSpec, context=None, last_rows=None, block=None):
    """gen_tucker_tensor (bench.hpp:83-95) on the device, fp64 flat column-major.
    last_rows=(offset, length): only that slab of the last mode (the global tensor's slab);
    block=(lo, ln): only that block."""
    import torch
    core = gaussian_flat(int(np.prod(mlranks)), seed.derived(0xC0DE), context)
    core_rm = core.view(*reversed([int(r) for r in mlranks]))
    fs = []
    for n, (i, r) in enumerate(zip(dims, mlranks)):
        a = gaussian_flat(int(i) * int(r), gen_factor_seed(seed, n), context).view(int(r), int(i)).t()
        fs.append(_rows(a, n, len(dims), last_rows, block))
    return _colmajor_einsum(core_rm, fs)


def gen_cp_device(dims, rank: int, seed: SeedSpec, uniform: bool = True, context=None, last_rows=None, block=None):
    """gen_cp_tensor (bench.hpp:56-80) with U(0,1) (or Gaussian) factors, fp64 flat column-major.
    last_rows=(offset, length): only that slab of the last mode."""
    import torch
    fs = []
    for n, i in enumerate(dims):
        if uniform:
            a = torch.from_numpy(uniform_matrix(int(i), rank, gen_factor_seed(seed, n))).cuda()
        else:
            a = gaussian_flat(int(i) * rank, gen_factor_seed(seed, n), context).view(rank, int(i)).t()
        fs.append(_rows(a, n, len(dims), last_rows, block))
    order = len(dims)
    eye = torch.zeros([rank] * order, dtype=torch.float64, device="cuda")
    idx = torch.arange(rank, device="cuda")
    eye[tuple([idx] * order)] = 1.0
    return _colmajor_einsum(eye, fs)


def add_noise_device(y, snr_db: float, seed: SeedSpec, abs_noise: bool = False, context=None, offset: int = 0,
                     all_sum=None):
    """add_noise (bench.hpp:100-112): sigma = ||Y|| / (||E|| 10^(snr/20)), Y + sigma E (in place).
    For a slab of a global tensor: `offset` = its first global flat index (noise drawn at the
    global indices) and `all_sum` sums the squared norms over the ranks holding the slabs."""
    import torch
    if np.isinf(snr_db) and snr_db > 0:
        return y
    e = gaussian_flat(y.numel(), seed.derived(0x7015E), context, offset=offset)
    if abs_noise:
        e.abs_()
    ysq = _sumsq(y)
    esq = _sumsq(e)
    if all_sum is not None:
        ysq, esq = all_sum(ysq), all_sum(esq)
    ny, ne = float(np.sqrt(ysq)), float(np.sqrt(esq))
    if ny <= 0 or ne <= 0:
        raise _lib.TenkitError("tenkit: add_noise: zero tensor input")
    sigma = ny / (ne * 10.0 ** (snr_db / 20.0))
    y.add_(e, alpha=sigma)
    del e
    return y


def _sumsq(x) -> float:
    """sum of squares in fp64 (chunked: BLAS dot takes 32-bit lengths)."""
    import torch
    n, tot, step = x.numel(), 0.0, 1 << 30
    for a in range(0, n, step):
        c = x[a:a + step]
        tot += float(torch.dot(c, c).item())
    return tot


def bench_seeds(seed: int = 0, d: int = 0, s: int = 0, run: int = 0):
    """run_experiment's seed derivation (bench.hpp:588,604-606): (data_seed, alg_seed)."""
    root = SeedSpec(seed, 0)
    return root.derived(0xDA7A, (d * 1000 + s) * 1000 + run), root.derived(0xA16D, run)


def generate(cfg: dict, context=None, slab=None, all_sum=None):
    """Observation Y (fp64 flat column-major CUDA tensor) of a benchmark config dict.
    slab=(offset, length): only that slab of the last mode of the global tensor cfg["dims"]
    (blockwise generation on the device: the slabs of all ranks concatenate to exactly the
    tensor a single generate() call produces, noise scale from norms summed by `all_sum`)."""
    data_seed, _ = bench_seeds(cfg.get("seed", 0))
    dims = [int(d) for d in cfg["dims"]]
    if cfg["gen"] == "tucker":
        y = gen_tucker_device(dims, cfg["mlrank"], data_seed, context, last_rows=slab)
    else:
        y = gen_cp_device(dims, cfg["cp_rank"], data_seed, uniform=cfg["gen"] == "cp_uniform", context=context,
                          last_rows=slab)
    offset = int(slab[0]) * int(np.prod(dims[:-1])) if slab is not None else 0
    return add_noise_device(y, cfg["snr"], data_seed.derived(0xAD0), abs_noise=cfg.get("abs_noise", False),
                            context=context, offset=offset, all_sum=all_sum)


def generate_as(cfg: dict, dtype, context=None, slab=None, all_sum=None, chunk_elems: int = 1 << 28,
                full_sigma: bool = False, block=None):
    """generate() straight into `dtype` (e.g. torch.float32) with bounded fp64 temporaries:
    the tensor (or this rank's last-mode slab) is built in chunks of the last mode, twice
    (pass 1: the norms of Y and E for sigma; pass 2: Y + sigma E rounded to dtype), every
    entry drawn at its global index. Same values as generate(...).to(dtype) up to the
    rounding of the chunked contractions; needed for cfg 3/4 (55 / 32 GB fp32) where the
    fp64 tensor and noise would not fit next to each other. full_sigma: materialise only
    `slab` but take the noise scale from the whole tensor (a bounded sample of it).
    block=(lo, ln): this rank's block of a BlockGrid instead of a slab (dist.GridPlan.block);
    the blocks of all ranks tile exactly the tensor generate() produces."""
    import torch
    dims = [int(d) for d in cfg["dims"]]
    if block is not None:
        if slab is not None or full_sigma:
            raise _lib.TenkitError("tenkit: generate: block excludes slab / full_sigma")
        blo, bln = [int(x) for x in block[0]], [int(x) for x in block[1]]
        slab = (blo[-1], bln[-1])
    off0, ln = (int(slab[0]), int(slab[1])) if slab is not None else (0, dims[-1])
    S = int(np.prod(dims[:-1])) if block is None else int(np.prod(bln[:-1]))
    per = max(1, int(chunk_elems) // S)
    data_seed, _ = bench_seeds(cfg.get("seed", 0))
    nseed = data_seed.derived(0xAD0).derived(0x7015E)
    abs_noise = cfg.get("abs_noise", False)
    noisy = not (np.isinf(cfg["snr"]) and cfg["snr"] > 0)

    def sub(a, b):  # the block restricted to rows [a, b) of the last mode
        return (blo[:-1] + [a], bln[:-1] + [b - a]) if block is not None else None

    def clean(a, b):  # rows [a, b) of the last mode (global indices)
        if cfg["gen"] == "tucker":
            return gen_tucker_device(dims, cfg["mlrank"], data_seed, context, last_rows=(a, b - a), block=sub(a, b))
        return gen_cp_device(dims, cfg["cp_rank"], data_seed, uniform=cfg["gen"] == "cp_uniform", context=context,
                             last_rows=(a, b - a), block=sub(a, b))

    def noise(a, b):
        if block is not None:
            e = gaussian_block(dims, *sub(a, b), nseed, context)
        else:
            e = gaussian_flat((b - a) * S, nseed, context, offset=a * S)
        return e.abs_() if abs_noise else e

    out = torch.empty(S * ln, dtype=dtype, device="cuda")
    ysq = esq = 0.0
    sigma = 0.0
    if noisy:
        n0, n1 = (0, dims[-1]) if full_sigma else (off0, off0 + ln)
        for a in range(n0, n1, per):
            b = min(a + per, n1)
            ysq += _sumsq(clean(a, b))
            esq += _sumsq(noise(a, b))
        if all_sum is not None:
            ysq, esq = all_sum(ysq), all_sum(esq)
        if ysq <= 0 or esq <= 0:
            raise _lib.TenkitError("tenkit: add_noise: zero tensor input")
        sigma = float(np.sqrt(ysq)) / (float(np.sqrt(esq)) * 10.0 ** (cfg["snr"] / 20.0))
    for a in range(off0, off0 + ln, per):
        b = min(a + per, off0 + ln)
        y = clean(a, b)
        if noisy:
            y.add_(noise(a, b), alpha=sigma)
        out[(a - off0) * S:(b - off0) * S] = y.to(dtype)
        del y
    return out
