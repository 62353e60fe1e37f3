// ttm.cu — the Y-streaming multilinear contraction kernels (sm_100a).
//
// Replaces the reference's ttm / ttm_all / unfold_times hot loop (tensor.hpp:151-209,
// driven from rand_tucker_2i at tucker.hpp:153,159,166). Y is read from HBM exactly once
// per pass: the first-stage kernel (ttm_mmajor_kernel) streams (P x K) column tiles of the
// (P, K, Q) slab view through a STAGES-deep ring of bulk-async copies (TMA engine,
// mbarrier complete_tx), contiguous along the fastest mode, while 8 consumer warps
// contract each tile against the resident factor chunk with fp32 FFMA (fp32-accurate,
// never TF32/BF16 — SURVEY App. B shows single-pass TF32 flips the sign rule).
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "kernels.cuh"

namespace tkb {

namespace {

template <typename T, int N>
struct Vec;
template <>
struct Vec<float, 4> {
    using type = float4;
};
template <>
struct Vec<float, 2> {
    using type = float2;
};
template <>
struct Vec<float, 1> {
    using type = float;
};
template <>
struct Vec<double, 2> {
    using type = double2;
};
template <>
struct Vec<double, 1> {
    using type = double;
};

template <typename T, int N>
__device__ __forceinline__ void load_vec(const T* p, T (&v)[N]) {
    using V = typename Vec<T, N>::type;
    const V x = *reinterpret_cast<const V*>(p);
    const T* xs = reinterpret_cast<const T*>(&x);
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = xs[i];
}
template <typename T, int N>
__device__ __forceinline__ void store_vec(T* p, const T (&v)[N]) {
    using V = typename Vec<T, N>::type;
    V x;
    T* xs = reinterpret_cast<T*>(&x);
#pragma unroll
    for (int i = 0; i < N; ++i) xs[i] = v[i];
    *reinterpret_cast<V*>(p) = x;
}

constexpr int kConsumers = 256;  // 8 consumer warps
constexpr int kBK = 16;          // K columns per pipeline stage
constexpr int kStages = 3;

template <typename T, int R>
struct MMajorCfg {
    static constexpr int R4 = (R + 3) / 4 * 4;
    // rows per thread: 128-bit vectors while the accumulator tile stays <= 128 registers
    static constexpr int TM = sizeof(T) == 4 ? (R <= 32 ? 4 : 2) : (R <= 32 ? 2 : 1);
    static constexpr int BM = kConsumers * TM;
    static constexpr size_t smem = size_t(kStages) * kBK * (BM + R4) * sizeof(T) + 2 * kStages * sizeof(uint64_t);
};

// out[p + r*P + q*P*cols] = sum_k in[p + k*P + q*P*K] * up[k*R4 + r]
template <typename T, int R>
__global__ void __launch_bounds__(kConsumers + 32, 1)
    ttm_mmajor_kernel(const T* __restrict__ in, const T* __restrict__ up, T* __restrict__ out, int64_t P,
                      int64_t K, int cols, int64_t tiles_p, int64_t Q, int64_t kchunk) {
    using Cfg = MMajorCfg<T, R>;
    constexpr int R4 = Cfg::R4, TM = Cfg::TM, BM = Cfg::BM;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    T* sY = reinterpret_cast<T*>(smem_raw);  // [kStages][kBK][BM]
    T* sU = sY + kStages * kBK * BM;          // [kStages][kBK][R4]
    uint64_t* full = reinterpret_cast<uint64_t*>(sU + kStages * kBK * R4);
    uint64_t* empty = full + kStages;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    // block -> (row tile, slab q, K split ks); split ks writes its own partial output
    const int64_t tq = tiles_p * Q;
    const int64_t ks = blockIdx.x / tq;
    const int64_t q = (blockIdx.x % tq) / tiles_p;
    const int64_t p0 = (blockIdx.x % tiles_p) * BM;
    const int rows = static_cast<int>(lmin(BM, P - p0));
    const int64_t kbeg = ks * kchunk;
    const int64_t klen = lmin(kchunk, K - kbeg);
    const T* base = in + q * P * K + kbeg * P + p0;
    up += kbeg * R4;
    out += ks * P * cols * Q;
    const int nk = static_cast<int>((klen + kBK - 1) / kBK);

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumers / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == kConsumers / 32) {  // producer warp: one lane drives the bulk-copy engine
        if (lane == 0) {
            for (int kc = 0; kc < nk; ++kc) {
                const int s = kc % kStages;
                const uint32_t ph = (kc / kStages) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                const int64_t k0 = int64_t(kc) * kBK;
                const int kn = static_cast<int>(lmin(kBK, klen - k0));
                const uint32_t ybytes = uint32_t(rows) * sizeof(T);
                mbar_arrive_expect_tx(&full[s], ybytes * kn + uint32_t(kn) * R4 * sizeof(T));
                for (int kk = 0; kk < kn; ++kk)
                    bulk_g2s(sY + (s * kBK + kk) * BM, base + (k0 + kk) * P, ybytes, &full[s]);
                bulk_g2s(sU + s * kBK * R4, up + k0 * R4, uint32_t(kn) * R4 * sizeof(T), &full[s]);
            }
        }
        return;
    }

    T acc[TM][R];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int r = 0; r < R; ++r) acc[i][r] = T(0);

    auto body = [&](const T* yrow, const T* urow) {
        T y[TM];
        load_vec<T, TM>(yrow, y);
#pragma unroll
        for (int r4 = 0; r4 < R4; r4 += 4) {
            T u[4];
            if constexpr (sizeof(T) == 4) {
                load_vec<T, 4>(urow + r4, u);
            } else {
                T a[2], b[2];
                load_vec<T, 2>(urow + r4, a);
                load_vec<T, 2>(urow + r4 + 2, b);
                u[0] = a[0], u[1] = a[1], u[2] = b[0], u[3] = b[1];
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (r4 + j < R)
#pragma unroll
                    for (int i = 0; i < TM; ++i) acc[i][r4 + j] = fma(y[i], u[j], acc[i][r4 + j]);
        }
    };

    for (int kc = 0; kc < nk; ++kc) {
        const int s = kc % kStages;
        const uint32_t ph = (kc / kStages) & 1;
        mbar_wait(&full[s], ph);
        const int kn = static_cast<int>(lmin(kBK, klen - int64_t(kc) * kBK));
        const T* ys = sY + s * kBK * BM + tid * TM;
        const T* us = sU + s * kBK * R4;
        if (kn == kBK) {
#pragma unroll
            for (int kk = 0; kk < kBK; ++kk) body(ys + kk * BM, us + kk * R4);
        } else {
            for (int kk = 0; kk < kn; ++kk) body(ys + kk * BM, us + kk * R4);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    }

    if (tid * TM < rows) {
        T* o = out + q * P * cols + p0 + tid * TM;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r < cols) {
                T v[TM];
#pragma unroll
                for (int i = 0; i < TM; ++i) v[i] = acc[i][r];
                store_vec<T, TM>(o + int64_t(r) * P, v);
            }
        }
    }
}

// Mode-0 contraction (P == 1): in is (K x A) column-major, K contiguous.
// out[r + a*cols] = sum_k in[k + a*K] * up[k*R4 + r] over this block's K range.
// A 128-column x 32-k tile is read with full-line loads (each thread one column) and
// transposed through shared memory; thread (q, g) then owns columns 4q..4q+3 and the
// r-quads g, g+4, ... so every k costs one 128-bit load of Y and one broadcast 128-bit
// load of U per 16 FMAs.
constexpr int kKcBA = 128;
template <typename T>
__host__ __device__ constexpr int kc_bk() { return sizeof(T) == 4 ? 32 : 16; }
template <typename T, int R>
__global__ void __launch_bounds__(128) ttm_kcontig_kernel(const T* __restrict__ in, const T* __restrict__ up,
                                                           T* __restrict__ out, int64_t K, int64_t A, int cols,
                                                           int64_t tiles_a, int64_t kchunk) {
    constexpr int R4 = (R + 3) / 4 * 4;
    constexpr int NP = (R4 + 15) / 16;  // r-passes of 16 (4 groups x 4)
    constexpr int kKcBK = kc_bk<T>();
    __shared__ __align__(16) T sT[kKcBK][kKcBA + 4];
    __shared__ __align__(16) T sU[kKcBK * R4];
    const int tid = threadIdx.x, q = tid & 31, g = tid >> 5;
    const int64_t a0 = (blockIdx.x % tiles_a) * kKcBA;
    const int64_t ks = blockIdx.x / tiles_a;
    const int64_t kbeg = ks * kchunk, kend = lmin(K, kbeg + kchunk);
    out += ks * int64_t(cols) * A;
    T acc[NP][4][4];
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int s = 0; s < 4; ++s) acc[p][c][s] = T(0);
    const int64_t acol = a0 + tid;
    const bool vec = (K % 4 == 0) && (reinterpret_cast<uintptr_t>(in) % 16 == 0);
    for (int64_t k0 = kbeg; k0 < kend; k0 += kKcBK) {
        const int kn = static_cast<int>(lmin(kKcBK, kend - k0));
        if (acol < A) {
            const T* src = in + acol * K + k0;
            if (vec && kn == kKcBK) {
#pragma unroll
                for (int v = 0; v < kKcBK; v += 16 / int(sizeof(T))) {
                    T tmp[16 / sizeof(T)];
                    load_vec<T, 16 / sizeof(T)>(src + v, tmp);
#pragma unroll
                    for (int e = 0; e < int(16 / sizeof(T)); ++e) sT[v + e][tid] = tmp[e];
                }
            } else {
                for (int kk = 0; kk < kKcBK; ++kk) sT[kk][tid] = kk < kn ? src[kk] : T(0);
            }
        } else {
            for (int kk = 0; kk < kKcBK; ++kk) sT[kk][tid] = T(0);
        }
        for (int i = tid; i < kKcBK * R4; i += 128) sU[i] = (i / R4 < kn) ? up[(k0 + i / R4) * R4 + i % R4] : T(0);
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < kKcBK; ++kk) {
            T y[4];
            if constexpr (sizeof(T) == 4) {
                load_vec<T, 4>(&sT[kk][4 * q], y);
            } else {
                T a2[2], b2[2];
                load_vec<T, 2>(&sT[kk][4 * q], a2);
                load_vec<T, 2>(&sT[kk][4 * q + 2], b2);
                y[0] = a2[0], y[1] = a2[1], y[2] = b2[0], y[3] = b2[1];
            }
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const int rb = 16 * p + 4 * g;
                if (rb < R4) {
                    T u[4];
                    if constexpr (sizeof(T) == 4) {
                        load_vec<T, 4>(&sU[kk * R4 + rb], u);
                    } else {
                        T a2[2], b2[2];
                        load_vec<T, 2>(&sU[kk * R4 + rb], a2);
                        load_vec<T, 2>(&sU[kk * R4 + rb + 2], b2);
                        u[0] = a2[0], u[1] = a2[1], u[2] = b2[0], u[3] = b2[1];
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int s2 = 0; s2 < 4; ++s2) acc[p][c][s2] = fma(y[c], u[s2], acc[p][c][s2]);
                }
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int64_t a = a0 + 4 * q + c;
        if (a < A)
#pragma unroll
            for (int p = 0; p < NP; ++p)
#pragma unroll
                for (int s2 = 0; s2 < 4; ++s2) {
                    const int r = 16 * p + 4 * g + s2;
                    if (r < cols) out[r + a * cols] = acc[p][c][s2];
                }
    }
}

// Shapes the tiled kernels do not take (P > 1 small or not a multiple of 4, e.g. the core
// contraction of a permuted X): CTA (q, 32-row block of p); lane = p, the 8 warps split K
// into contiguous chunks; each thread keeps the R outputs of its p in registers, reading x
// coalesced along p and the U row as warp-broadcast vectors; the chunks are summed in fixed
// order through shared memory.
template <typename T, int R>
__global__ void __launch_bounds__(256) ttm_smallp_kernel(const T* __restrict__ in, const T* __restrict__ up,
                                                         T* __restrict__ out, int64_t P, int64_t K, int cols,
                                                         int stride) {
    constexpr int RC = 16;  // outputs per reduction round
    __shared__ T red[8][RC][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t q = blockIdx.x;
    const int64_t p = int64_t(blockIdx.y) * 32 + lane;
    const bool live = p < P;
    // split-K over gridDim.z: this CTA's K range, split into 8 warp chunks; partial z goes to
    // out + z * (P * cols * gridDim.x)
    const int64_t kz = (K + gridDim.z - 1) / gridDim.z;
    const int64_t kz0 = int64_t(blockIdx.z) * kz, kz1 = kz0 + kz < K ? kz0 + kz : K;
    const int64_t kc = (kz1 - kz0 + 7) / 8;
    const int64_t k0 = kz0 + warp * kc, k1 = k0 + kc < kz1 ? k0 + kc : kz1;
    out += int64_t(blockIdx.z) * P * cols * gridDim.x;
    const T* src = in + (live ? p : 0) + q * P * K;
    T acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = T(0);
    constexpr int KU = 8;  // x loads in flight per thread
    int64_t k = k0;
    for (; k + KU <= k1; k += KU) {
        T x[KU];
#pragma unroll
        for (int e = 0; e < KU; ++e) x[e] = live ? src[(k + e) * P] : T(0);
#pragma unroll
        for (int e = 0; e < KU; ++e) {
            const T* u = up + (k + e) * stride;
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = fma(x[e], u[r], acc[r]);
        }
    }
    for (; k < k1; ++k) {
        const T x = live ? src[k * P] : T(0);
        const T* u = up + k * stride;
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma(x, u[r], acc[r]);
    }
#pragma unroll
    for (int rc = 0; rc < R; rc += RC) {
#pragma unroll
        for (int e = 0; e < RC; ++e)
            if (rc + e < R) red[warp][e][lane] = acc[rc + e];
        __syncthreads();
        for (int t = threadIdx.x; t < RC * 32; t += 256) {
            const int e = t >> 5, l = t & 31;
            const int64_t pp = int64_t(blockIdx.y) * 32 + l;
            if (rc + e < cols && pp < P) {
                T v = red[0][e][l];
#pragma unroll
                for (int w = 1; w < 8; ++w) v += red[w][e][l];
                out[pp + int64_t(rc + e) * P + q * P * cols] = v;
            }
        }
        __syncthreads();
    }
}

// fixed-order sum of split-K partials: out[i] = sum_s part[s*n + i]
template <typename T>
__global__ void splitk_reduce_kernel(const T* __restrict__ part, T* __restrict__ out, int64_t n, int splits) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        T acc = part[i];
        for (int sidx = 1; sidx < splits; ++sidx) acc += part[sidx * n + i];
        out[i] = acc;
    }
}

template <typename T, int R>
void dispatch_ttm(const T* in, const T* up, T* out, int64_t P, int64_t K, int64_t Q, int cols, cudaStream_t s,
                  T* work, int64_t work_elems, int* launches) {
    using Cfg = MMajorCfg<T, R>;
    const bool aligned = (reinterpret_cast<uintptr_t>(in) % 16 == 0) && (reinterpret_cast<uintptr_t>(up) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    if (P % 4 == 0 && P >= 64 && aligned) {
        static bool attr = false;
        if (!attr) {
            TK_CUDA(cudaFuncSetAttribute(ttm_mmajor_kernel<T, R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::smem)));
            attr = true;
        }
        const int64_t tiles_p = (P + Cfg::BM - 1) / Cfg::BM;
        const int64_t tiles = tiles_p * Q;
        // split K when the row tiles cannot fill 2 waves of the 148 SMs
        int64_t splits = 1;
        if (tiles < 2 * 148 && K >= 8 * kBK && work) {
            splits = std::min<int64_t>((2 * 148 + tiles - 1) / tiles, K / (4 * kBK));
            while (splits > 1 && splits * P * cols * Q > work_elems) --splits;
        }
        const int64_t kchunk = ((K + splits - 1) / splits + kBK - 1) / kBK * kBK;
        splits = (K + kchunk - 1) / kchunk;
        const int64_t grid = tiles * splits;
        require(grid < (int64_t(1) << 31), "ttm: grid too large");
        T* dst = splits > 1 ? work : out;
        TK_MAXSMEM((ttm_mmajor_kernel<T, R>));
        ttm_mmajor_kernel<T, R><<<static_cast<unsigned>(grid), kConsumers + 32, Cfg::smem, s>>>(in, up, dst, P, K, cols,
                                                                                                tiles_p, Q, kchunk);
        if (splits > 1) {
            TK_LAUNCH_CHECK();
            const int64_t n = P * cols * Q;
            TK_MAXSMEM((splitk_reduce_kernel<T>));
            splitk_reduce_kernel<T><<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(
                work, out, n, static_cast<int>(splits));
            if (launches) ++*launches;
        }
    } else if (P == 1) {
        const int64_t tiles_a = (Q + kKcBA - 1) / kKcBA;
        int64_t splits = 1;
        constexpr int bk = kc_bk<T>();
        if (tiles_a < 4 * 148 && K >= 4 * bk && work) {
            splits = std::min<int64_t>((4 * 148 + tiles_a - 1) / tiles_a, K / (2 * bk));
            while (splits > 1 && splits * cols * Q > work_elems) --splits;
        }
        const int64_t kchunk = ((K + splits - 1) / splits + bk - 1) / bk * bk;
        splits = (K + kchunk - 1) / kchunk;
        T* dst = splits > 1 ? work : out;
        TK_MAXSMEM((ttm_kcontig_kernel<T, R>));
        ttm_kcontig_kernel<T, R><<<static_cast<unsigned>(tiles_a * splits), 128, 0, s>>>(in, up, dst, K, Q, cols,
                                                                                         tiles_a, kchunk);
        if (splits > 1) {
            TK_LAUNCH_CHECK();
            const int64_t n = int64_t(cols) * Q;
            TK_MAXSMEM((splitk_reduce_kernel<T>));
            splitk_reduce_kernel<T><<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(
                work, out, n, static_cast<int>(splits));
            if (launches) ++*launches;
        }
    } else {
        require(Q < (int64_t(1) << 31) && (P + 31) / 32 < 65536, "ttm: extent too large");
        const int64_t ctas = Q * ((P + 31) / 32);
        // split K when the (q, p-block) CTAs cannot fill 2 waves: >= 128 k per split
        int64_t splits = 1;
        if (ctas < 2 * 148 && K >= 256 && work) {
            splits = std::min<int64_t>({(2 * 148 + ctas - 1) / ctas, K / 128, 64});
            while (splits > 1 && splits * P * cols * Q > work_elems) --splits;
        }
        T* dst = splits > 1 ? work : out;
        TK_MAXSMEM((ttm_smallp_kernel<T, R>));
        ttm_smallp_kernel<T, R><<<dim3(static_cast<unsigned>(Q), static_cast<unsigned>((P + 31) / 32),
                                       static_cast<unsigned>(splits)), 256, 0, s>>>(in, up, dst, P, K, cols,
                                                                                   pack_stride(cols));
        if (splits > 1) {
            TK_LAUNCH_CHECK();
            const int64_t n = P * cols * Q;
            TK_MAXSMEM((splitk_reduce_kernel<T>));
            splitk_reduce_kernel<T><<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(
                work, out, n, static_cast<int>(splits));
            if (launches) ++*launches;
        }
    }
    TK_LAUNCH_CHECK();
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void pack_factor_kernel(const double* __restrict__ u, int64_t ld, int64_t rows, int cols, int stride,
                                   T* __restrict__ up) {
    const int64_t n = rows * stride;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t k = i / stride;
        const int r = static_cast<int>(i % stride);
        up[i] = r < cols ? static_cast<T>(u[k + r * ld]) : T(0);
    }
}

__global__ void gaussian_colmajor_kernel(double* __restrict__ out, uint64_t n, uint64_t key) {
    for (uint64_t pr = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; 2 * pr < n; pr += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = 2 * pr;
        const double u1 = counter_unit(key, i), u2 = counter_unit(key, i + 1);
        const double r = sqrt(-2.0 * log(u1));
        const double ang = 6.283185307179586476925287 * u2;
        out[i] = r * cos(ang);
        if (i + 1 < n) out[i + 1] = r * sin(ang);
    }
}


// out[t] = normal_at(key, off + t), t < n: a window of gaussian_tensor (random.hpp:124-138)
// at an arbitrary flat offset (a rank's slab of a globally indexed tensor)
__global__ void gaussian_fill_kernel(double* __restrict__ out, uint64_t n, uint64_t off, uint64_t key) {
    const uint64_t first = off >> 1, last = (off + n - 1) >> 1;
    for (uint64_t pr = first + blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; pr <= last;
         pr += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t i = 2 * pr;
        const double u1 = counter_unit(key, i), u2 = counter_unit(key, i + 1);
        const double r = sqrt(-2.0 * log(u1));
        const double ang = 6.283185307179586476925287 * u2;
        if (i >= off && i < off + n) out[i - off] = r * cos(ang);
        if (i + 1 >= off && i + 1 < off + n) out[i + 1 - off] = r * sin(ang);
    }
}

// Z (fp64, ldz) = unfold(X, n) Omega for X viewed as (B, I, A): Z[i, r] = sum over
// k = b + a B of X[b + i B + a B I] Omega[k, r] (tensor.hpp:195-209 unfold_times), without
// materialising the unfolding. CTA tile 32 rows x 32 columns, split-K over blockIdx.z into
// fp64 partials summed in fixed order by sketch_reduce_kernel; fp64 accumulation.
template <typename T>
__global__ void __launch_bounds__(256) sketch_kernel(const T* __restrict__ x, int B, int64_t I, int A,
                                                     const T* __restrict__ om, int stride, int rn, int kchunk,
                                                     double* __restrict__ part) {
    __shared__ double xs[64][33];
    __shared__ double os[64][33];
    const int tid = threadIdx.x, ti = tid & 31, tr = tid >> 5;
    const int64_t i0 = int64_t(blockIdx.x) * 32;
    const int r0 = blockIdx.y * 32;
    const int K = B * A;
    const int k0 = blockIdx.z * kchunk, k1 = min(K, k0 + kchunk);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int kk = k0; kk < k1; kk += 64) {
        for (int e = tid; e < 64 * 32; e += 256) {
            // coalesced: consecutive threads walk the contiguous index (i when B == 1, else b)
            const int kl = B == 1 ? (e >> 5) : (e & 63), il = B == 1 ? (e & 31) : (e >> 6);
            const int k = kk + kl;
            const int64_t i = i0 + il;
            double v = 0.0;
            if (k < k1 && i < I) {
                const int b = k % B, a = k / B;
                v = static_cast<double>(x[b + i * B + int64_t(a) * B * I]);
            }
            xs[kl][il] = v;
        }
        for (int e = tid; e < 64 * 32; e += 256) {
            const int kl = e >> 5, rl = e & 31;
            const int k = kk + kl, r = r0 + rl;
            os[kl][rl] = (k < k1 && r < rn) ? static_cast<double>(om[int64_t(k) * stride + r]) : 0.0;
        }
        __syncthreads();
        const int kn = min(64, k1 - kk);
        for (int k = 0; k < kn; ++k) {
            const double xv = xs[k][ti];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = fma(xv, os[k][tr * 4 + j], acc[j]);
        }
        __syncthreads();
    }
    const int64_t i = i0 + ti;
    if (i < I)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int r = r0 + tr * 4 + j;
            if (r < rn) part[(int64_t(blockIdx.z) * rn + r) * I + i] = acc[j];
        }
}

// The same with one CTA covering ALL rn columns (rn <= 64) of its 32 rows: thread (lane = row,
// warp = column group of CG = ceil(rn / 8) columns). X is staged once per row tile (the 32-column
// tiles above stage it once per column tile and leave 24 of 64 columns idle at rn = 40), and a
// k step costs 1 + CG shared loads for CG FMAs. KT = k per staging round (32 when CG > 4, so the
// two staging buffers stay inside the static shared-memory limit).
template <typename T, int CG, int KT>
__global__ void __launch_bounds__(256) sketch_wide_kernel(const T* __restrict__ x, int B, int64_t I, int A,
                                                          const T* __restrict__ om, int stride, int rn, int kchunk,
                                                          double* __restrict__ part) {
    constexpr int NC = 8 * CG;
    __shared__ double xs[KT][33];
    __shared__ double os[KT][NC + 1];
    const int tid = threadIdx.x, ti = tid & 31, tr = tid >> 5;
    const int64_t i0 = int64_t(blockIdx.x) * 32;
    const int K = B * A;
    const int k0 = blockIdx.z * kchunk, k1 = min(K, k0 + kchunk);
    double acc[CG];
#pragma unroll
    for (int j = 0; j < CG; ++j) acc[j] = 0.0;
    for (int kk = k0; kk < k1; kk += KT) {
        for (int e = tid; e < KT * 32; e += 256) {
            // coalesced: consecutive threads walk the contiguous index (i when B == 1, else b)
            const int kl = B == 1 ? (e >> 5) : (e % KT), il = B == 1 ? (e & 31) : (e / KT);
            const int k = kk + kl;
            const int64_t i = i0 + il;
            double v = 0.0;
            if (k < k1 && i < I) {
                const int b = k % B, a = k / B;
                v = static_cast<double>(x[b + i * B + int64_t(a) * B * I]);
            }
            xs[kl][il] = v;
        }
        for (int e = tid; e < KT * NC; e += 256) {
            const int kl = e / NC, rl = e % NC;
            const int k = kk + kl;
            os[kl][rl] = (k < k1 && rl < rn) ? static_cast<double>(om[int64_t(k) * stride + rl]) : 0.0;
        }
        __syncthreads();
        const int kn = min(KT, k1 - kk);
        for (int k = 0; k < kn; ++k) {
            const double xv = xs[k][ti];
#pragma unroll
            for (int j = 0; j < CG; ++j) acc[j] = fma(xv, os[k][tr * CG + j], acc[j]);
        }
        __syncthreads();
    }
    const int64_t i = i0 + ti;
    if (i < I)
#pragma unroll
        for (int j = 0; j < CG; ++j) {
            const int r = tr * CG + j;
            if (r < rn) part[(int64_t(blockIdx.z) * rn + r) * I + i] = acc[j];
        }
}

__global__ void sketch_reduce_kernel(const double* __restrict__ part, int64_t I, int rn, int S, double* __restrict__ z,
                                     int64_t ldz) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < I * rn; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = t % I, r = t / I;
        double v = 0.0;
        for (int sidx = 0; sidx < S; ++sidx) v += part[(int64_t(sidx) * rn + r) * I + i];
        z[i + r * ldz] = v;
    }
}

// out[i + c*I] = x[b + i*B + a*B*I], c = b + a*B: the mode-n unfolding of a (B, I, A) view
template <typename T>
__global__ void unfold_kernel(const T* __restrict__ x, int64_t B, int64_t I, int64_t A, T* __restrict__ out) {
    const int64_t n = B * I * A;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t b = t % B, i = (t / B) % I, a = t / (B * I);
        out[i + (b + a * B) * I] = x[t];
    }
}

template <typename T>
__global__ void gaussian_packed_kernel(T* __restrict__ out, int64_t rows, int cols, int stride, uint64_t key,
                                       int64_t row_off, int64_t rows_total) {
    const int64_t n = rows * stride;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = t / stride;
        const int j = static_cast<int>(t % stride);
        out[t] = j < cols ? static_cast<T>(normal_at_key(key, static_cast<uint64_t>(j * rows_total + row_off + c))) : T(0);
    }
}

template <typename T>
__global__ void gaussian_packed_map_kernel(T* __restrict__ out, int64_t rows, int cols, int stride, uint64_t key,
                                           RowMap map) {
    const int64_t n = rows * stride;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = t / stride;
        const int j = static_cast<int>(t % stride);
        int64_t g = 0, rem = c;
        for (int k = 0; k < map.nd; ++k) {
            const int64_t d = rem % map.lext[k];
            rem /= map.lext[k];
            g += (map.lo[k] + d) * map.gstride[k];
        }
        out[t] = j < cols ? static_cast<T>(normal_at_key(key, static_cast<uint64_t>(j * map.rows_total + g))) : T(0);
    }
}

struct PermDesc {
    int order;
    int64_t dims[8];     // standard extents
    int64_t sstride[8];  // storage stride of each (standard) mode
};

template <typename S, typename D>
__global__ void permute_cast_kernel(const S* __restrict__ in, D* __restrict__ out, int64_t n, PermDesc pd) {
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        int64_t rem = t, src = 0;
        for (int k = 0; k < pd.order; ++k) {
            src += (rem % pd.dims[k]) * pd.sstride[k];
            rem /= pd.dims[k];
        }
        out[t] = static_cast<D>(in[src]);
    }
}

template <typename S, typename D>
__global__ void cast2d_kernel(const S* __restrict__ in, int64_t ldi, D* __restrict__ out, int64_t ldo, int64_t rows,
                              int64_t cols) {
    const int64_t n = rows * cols;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = t % rows, j = t / rows;
        out[i + j * ldo] = static_cast<D>(in[i + j * ldi]);
    }
}

template <typename S, typename D>
__global__ void cast_kernel(const S* __restrict__ in, D* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = static_cast<D>(in[i]);
}

inline unsigned grid_for(int64_t n, int per = 256) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + per - 1) / per, 148 * 16)));
}

}  // namespace

template <typename T>
void launch_ttm(const T* in, const T* up, T* out, int64_t P, int64_t K, int64_t Q, int cols, cudaStream_t s,
                int* launches, T* work, int64_t work_elems) {
    require(cols >= 1 && cols <= kMaxRank, "ttm: factor column count must be in [1, 64]");
    require(P >= 1 && K >= 1 && Q >= 1, "ttm: empty slab view");
    if (launches) ++*launches;
    // kernel instantiations: exact 15/30 (bench configs) else the next multiple of 4
    if (cols == 15) return dispatch_ttm<T, 15>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
    if (cols == 30) return dispatch_ttm<T, 30>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
    switch (pack_stride(cols)) {
        case 4: return dispatch_ttm<T, 4>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 8: return dispatch_ttm<T, 8>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 12: return dispatch_ttm<T, 12>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 16: return dispatch_ttm<T, 16>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 20: return dispatch_ttm<T, 20>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 24: return dispatch_ttm<T, 24>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 28: return dispatch_ttm<T, 28>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 32: return dispatch_ttm<T, 32>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 36: return dispatch_ttm<T, 36>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 40: return dispatch_ttm<T, 40>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 44: return dispatch_ttm<T, 44>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 48: return dispatch_ttm<T, 48>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 52: return dispatch_ttm<T, 52>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 56: return dispatch_ttm<T, 56>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        case 60: return dispatch_ttm<T, 60>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
        default: return dispatch_ttm<T, 64>(in, up, out, P, K, Q, cols, s, work, work_elems, launches);
    }
}

template <typename T>
void launch_pack_factor(const double* u, int64_t ld, int64_t rows, int cols, T* up, cudaStream_t s) {
    const int stride = pack_stride(cols);
    TK_MAXSMEM((pack_factor_kernel<T>));
    pack_factor_kernel<T><<<grid_for(rows * stride), 256, 0, s>>>(u, ld, rows, cols, stride, up);
    TK_LAUNCH_CHECK();
}

void launch_gaussian_fill(double* out, int64_t n, uint64_t offset, uint64_t key, cudaStream_t s) {
    if (n <= 0) return;
    TK_MAXSMEM((gaussian_fill_kernel));
    gaussian_fill_kernel<<<grid_for((n + 3) / 2), 256, 0, s>>>(out, uint64_t(n), offset, key);
    TK_LAUNCH_CHECK();
}

void launch_gaussian_colmajor(double* out, int64_t rows, int64_t cols, uint64_t key, cudaStream_t s) {
    const uint64_t n = uint64_t(rows) * uint64_t(cols);
    TK_MAXSMEM((gaussian_colmajor_kernel));
    gaussian_colmajor_kernel<<<grid_for(static_cast<int64_t>((n + 1) / 2)), 256, 0, s>>>(out, n, key);
    TK_LAUNCH_CHECK();
}


// Split-K factor of the sketch: the kernel is latency-bound per CTA (ncu at cfg 2: 0.35 waves,
// issue-bound), so K is split until the grid holds ~kSketchCtas CTAs (4 per SM), at most 64
// splits, at least 64 k per split. (cfg 4: I = 300, K = 8000 -> 42 splits instead of 16.)
static int sketch_split_cap(int64_t I, int rn) {
    static const int64_t target = [] {
        const char* e = std::getenv("TENKIT_SKETCH_CTAS");
        return e ? std::max<int64_t>(1, std::atoll(e)) : int64_t(4 * 148);
    }();
    const int64_t tiles = (I + 31) / 32;  // one CTA covers every column of its 32 rows (rn <= 64)
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, (target + tiles - 1) / tiles)));
}

int64_t sketch_work_elems(int64_t I, int rn) { return I * rn * sketch_split_cap(I, rn); }

template <typename T>
int launch_sketch_partials(const T* x, int64_t B, int64_t I, int64_t A, const T* om, int rn, double* work,
                           cudaStream_t s, int max_splits) {
    require(B * A < (int64_t(1) << 31), "unfold_times: unfolding too wide");
    const int K = static_cast<int>(B * A);
    const unsigned gx = static_cast<unsigned>((I + 31) / 32), gy = static_cast<unsigned>((rn + 31) / 32);
    int S = std::min(sketch_split_cap(I, rn), std::max(1, max_splits));
    S = std::max(1, std::min(S, (K + 63) / 64));
    const int kchunk = ((K + S - 1) / S + 63) / 64 * 64;
    S = (K + kchunk - 1) / kchunk;
    static const bool narrow = [] {  // A/B knob: the 32-column tiles
        const char* e = std::getenv("TENKIT_SKETCH_NARROW");
        return e && e[0] == '1';
    }();
    if (narrow || rn <= 32 || rn > 64) {  // (one 32-column tile already covers rn <= 32)
        TK_MAXSMEM((sketch_kernel<T>));
        sketch_kernel<T><<<dim3(gx, gy, S), 256, 0, s>>>(x, static_cast<int>(B), I, static_cast<int>(A), om, pack_stride(rn),
                                                         rn, kchunk, work);
        TK_LAUNCH_CHECK();
        return S;
    }
#define TK_SKETCH_CASE(CG, KT)                                                                                     \
    case CG:                                                                                                       \
        sketch_wide_kernel<T, CG, KT><<<dim3(gx, 1, S), 256, 0, s>>>(x, static_cast<int>(B), I, static_cast<int>(A), om, \
                                                                     pack_stride(rn), rn, kchunk, work);           \
        break;
    switch ((rn + 7) / 8) {
        TK_SKETCH_CASE(5, 32)
        TK_SKETCH_CASE(6, 32)
        TK_SKETCH_CASE(7, 32)
        TK_SKETCH_CASE(8, 32)
    }
#undef TK_SKETCH_CASE
    TK_LAUNCH_CHECK();
    return S;
}

template <typename T>
int launch_sketch(const T* x, int64_t B, int64_t I, int64_t A, const T* om, int rn, double* z, int64_t ldz, double* work,
                  cudaStream_t s) {
    const int S = launch_sketch_partials<T>(x, B, I, A, om, rn, work, s, 64);
    TK_MAXSMEM((sketch_reduce_kernel));
    sketch_reduce_kernel<<<grid_for(I * rn), 256, 0, s>>>(work, I, rn, S, z, ldz);
    TK_LAUNCH_CHECK();
    return 2;
}
template int launch_sketch_partials<float>(const float*, int64_t, int64_t, int64_t, const float*, int, double*,
                                           cudaStream_t, int);
template int launch_sketch_partials<double>(const double*, int64_t, int64_t, int64_t, const double*, int, double*,
                                            cudaStream_t, int);
template int launch_sketch<float>(const float*, int64_t, int64_t, int64_t, const float*, int, double*, int64_t, double*,
                                  cudaStream_t);
template int launch_sketch<double>(const double*, int64_t, int64_t, int64_t, const double*, int, double*, int64_t, double*,
                                   cudaStream_t);

template <typename T>
void launch_unfold(const T* x, int64_t B, int64_t I, int64_t A, T* out, cudaStream_t s) {
    TK_MAXSMEM((unfold_kernel<T>));
    unfold_kernel<T><<<grid_for(B * I * A), 256, 0, s>>>(x, B, I, A, out);
    TK_LAUNCH_CHECK();
}
template void launch_unfold<float>(const float*, int64_t, int64_t, int64_t, float*, cudaStream_t);
template void launch_unfold<double>(const double*, int64_t, int64_t, int64_t, double*, cudaStream_t);

template <typename T>
void launch_gaussian_packed(T* out, int64_t rows, int cols, uint64_t key, cudaStream_t s, int64_t row_off,
                            int64_t rows_total) {
    const int stride = pack_stride(cols);
    if (rows_total <= 0) rows_total = rows;
    TK_MAXSMEM((gaussian_packed_kernel<T>));
    gaussian_packed_kernel<T><<<grid_for(rows * stride), 256, 0, s>>>(out, rows, cols, stride, key, row_off, rows_total);
    TK_LAUNCH_CHECK();
}
template void launch_gaussian_packed<float>(float*, int64_t, int, uint64_t, cudaStream_t, int64_t, int64_t);
template void launch_gaussian_packed<double>(double*, int64_t, int, uint64_t, cudaStream_t, int64_t, int64_t);

template <typename T>
void launch_gaussian_packed_map(T* out, int64_t rows, int cols, uint64_t key, const RowMap& map, cudaStream_t s) {
    const int stride = pack_stride(cols);
    TK_MAXSMEM((gaussian_packed_map_kernel<T>));
    gaussian_packed_map_kernel<T><<<grid_for(rows * stride), 256, 0, s>>>(out, rows, cols, stride, key, map);
    TK_LAUNCH_CHECK();
}
void launch_gaussian_fill_map(double* out, int64_t n, uint64_t key, const RowMap& map, cudaStream_t s) {
    // stride 1, one column: out[c] = normal_at(key, 0 * rows_total + g(c))
    TK_MAXSMEM((gaussian_packed_map_kernel<double>));
    gaussian_packed_map_kernel<double><<<grid_for(n), 256, 0, s>>>(out, n, 1, 1, key, map);
    TK_LAUNCH_CHECK();
}
template void launch_gaussian_packed_map<float>(float*, int64_t, int, uint64_t, const RowMap&, cudaStream_t);
template void launch_gaussian_packed_map<double>(double*, int64_t, int, uint64_t, const RowMap&, cudaStream_t);

template <typename S, typename D>
void launch_cast(const S* in, D* out, int64_t n, cudaStream_t s) {
    TK_MAXSMEM((cast_kernel<S, D>));
    cast_kernel<S, D><<<grid_for(n), 256, 0, s>>>(in, out, n);
    TK_LAUNCH_CHECK();
}

template <typename S, typename D>
void launch_permute_cast(const S* in, D* out, int order, const int64_t* dims, const int* perm, cudaStream_t s) {
    require(order >= 1 && order <= 8, "permute: order must be in [1, 8]");
    PermDesc pd{};
    pd.order = order;
    int64_t n = 1, st = 1;
    for (int k = 0; k < order; ++k) {
        pd.dims[k] = dims[k];
        n *= dims[k];
    }
    for (int k = 0; k < order; ++k) {  // storage position k holds mode perm[k]
        pd.sstride[perm[k]] = st;
        st *= dims[perm[k]];
    }
    TK_MAXSMEM((permute_cast_kernel<S, D>));
    permute_cast_kernel<S, D><<<grid_for(n), 256, 0, s>>>(in, out, n, pd);
    TK_LAUNCH_CHECK();
}
template void launch_permute_cast<float, double>(const float*, double*, int, const int64_t*, const int*, cudaStream_t);
template void launch_permute_cast<double, double>(const double*, double*, int, const int64_t*, const int*, cudaStream_t);
template void launch_permute_cast<float, float>(const float*, float*, int, const int64_t*, const int*, cudaStream_t);

template <typename T>
void launch_splitk_reduce(const T* part, T* out, int64_t n, int splits, cudaStream_t s) {
    TK_MAXSMEM((splitk_reduce_kernel<T>));
    splitk_reduce_kernel<T><<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(
        part, out, n, splits);
    TK_LAUNCH_CHECK();
}
template void launch_splitk_reduce<float>(const float*, float*, int64_t, int, cudaStream_t);

template void launch_ttm<float>(const float*, const float*, float*, int64_t, int64_t, int64_t, int, cudaStream_t, int*,
                                float*, int64_t);
template void launch_ttm<double>(const double*, const double*, double*, int64_t, int64_t, int64_t, int, cudaStream_t,
                                 int*, double*, int64_t);
template void launch_pack_factor<float>(const double*, int64_t, int64_t, int, float*, cudaStream_t);
template void launch_pack_factor<double>(const double*, int64_t, int64_t, int, double*, cudaStream_t);
template <typename S, typename D>
void launch_cast2d(const S* in, int64_t ldi, D* out, int64_t ldo, int64_t rows, int64_t cols, cudaStream_t s) {
    TK_MAXSMEM((cast2d_kernel<S, D>));
    cast2d_kernel<S, D><<<grid_for(rows * cols), 256, 0, s>>>(in, ldi, out, ldo, rows, cols);
    TK_LAUNCH_CHECK();
}
template void launch_cast2d<float, double>(const float*, int64_t, double*, int64_t, int64_t, int64_t, cudaStream_t);
template void launch_cast2d<double, double>(const double*, int64_t, double*, int64_t, int64_t, int64_t, cudaStream_t);
template void launch_cast<float, double>(const float*, double*, int64_t, cudaStream_t);
template void launch_cast<double, float>(const double*, float*, int64_t, cudaStream_t);
template void launch_cast<double, double>(const double*, double*, int64_t, cudaStream_t);
template void launch_cast<float, float>(const float*, float*, int64_t, cudaStream_t);

}  // namespace tkb
