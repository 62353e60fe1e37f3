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
// out[r + a*cols] = sum_k in[k + a*K] * up[k*R4 + r]. Tiles are transposed through
// shared memory so the K-contiguous reads stay coalesced.
constexpr int kKcBA = 256;
template <typename T, int R>
__global__ void __launch_bounds__(256) ttm_kcontig_kernel(const T* __restrict__ in, const T* __restrict__ up,
                                                           T* __restrict__ out, int64_t K, int64_t A, int cols) {
    constexpr int R4 = (R + 3) / 4 * 4;
    constexpr int kKcBK = sizeof(T) == 4 ? 32 : 16;
    __shared__ T sT[kKcBK][kKcBA + 1];
    __shared__ __align__(16) T sU[kKcBK * R4];
    const int tid = threadIdx.x;
    const int64_t a0 = int64_t(blockIdx.x) * kKcBA;
    T acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = T(0);
    for (int64_t k0 = 0; k0 < K; k0 += kKcBK) {
        const int kn = static_cast<int>(lmin(kKcBK, K - k0));
        for (int idx = tid; idx < kKcBK * kKcBA; idx += 256) {
            const int kk = idx % kKcBK, c = idx / kKcBK;
            const int64_t a = a0 + c;
            sT[kk][c] = (a < A && kk < kn) ? in[(k0 + kk) + a * K] : T(0);
        }
        for (int i = tid; i < kKcBK * R4; i += 256) sU[i] = (i / R4 < kn) ? up[k0 * R4 + i] : T(0);
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < kKcBK; ++kk) {
            const T y = sT[kk][tid];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = fma(y, sU[kk * R4 + r], acc[r]);
        }
        __syncthreads();
    }
    const int64_t a = a0 + tid;
    if (a < A)
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (r < cols) out[r + a * cols] = acc[r];
}

// Any shape: one output element per thread.
template <typename T>
__global__ void ttm_generic_kernel(const T* __restrict__ in, const T* __restrict__ up, T* __restrict__ out,
                                   int64_t P, int64_t K, int64_t Q, int cols, int stride) {
    const int64_t n = P * cols * Q;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n; idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t p = idx % P;
        const int r = static_cast<int>((idx / P) % cols);
        const int64_t q = idx / (P * cols);
        const T* src = in + p + q * P * K;
        T acc = T(0);
        for (int64_t k = 0; k < K; ++k) acc = fma(src[k * P], up[k * stride + r], acc);
        out[idx] = acc;
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
        ttm_mmajor_kernel<T, R><<<static_cast<unsigned>(grid), kConsumers + 32, Cfg::smem, s>>>(in, up, dst, P, K, cols,
                                                                                                tiles_p, Q, kchunk);
        if (splits > 1) {
            TK_LAUNCH_CHECK();
            const int64_t n = P * cols * Q;
            splitk_reduce_kernel<T><<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0, s>>>(
                work, out, n, static_cast<int>(splits));
            if (launches) ++*launches;
        }
    } else if (P == 1) {
        const int64_t grid = (Q + kKcBA - 1) / kKcBA;
        ttm_kcontig_kernel<T, R><<<static_cast<unsigned>(grid), 256, 0, s>>>(in, up, out, K, Q, cols);
    } else {
        const int64_t n = P * cols * Q;
        const int64_t grid = std::min<int64_t>((n + 255) / 256, 148 * 32);
        ttm_generic_kernel<T><<<static_cast<unsigned>(grid), 256, 0, s>>>(in, up, out, P, K, Q, cols,
                                                                         pack_stride(cols));
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

// Z[i + j*ldz] = sum_c X[b + i*B + a*B*I] * omega_t[c*rn + j], c = b + a*B
template <typename T>
__global__ void __launch_bounds__(256) sketch_kernel(const T* __restrict__ x, int64_t B, int64_t I, int64_t A,
                                                     const double* __restrict__ omega_t, int rn, double* __restrict__ z,
                                                     int64_t ldz) {
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    __shared__ double red[8][kMaxRank];
    const int64_t W = B * A;
    for (int64_t i = blockIdx.x; i < I; i += gridDim.x) {
        double acc0 = 0.0, acc1 = 0.0;
        for (int64_t c = ty; c < W; c += 8) {
            const int64_t b = c % B, a = c / B;
            const double xv = static_cast<double>(x[b + i * B + a * B * I]);
            const double* om = omega_t + c * rn;
            if (tx < rn) acc0 = fma(xv, om[tx], acc0);
            if (tx + 32 < rn) acc1 = fma(xv, om[tx + 32], acc1);
        }
        red[ty][tx] = acc0;
        red[ty][tx + 32] = acc1;
        __syncthreads();
        if (ty == 0) {
            for (int j = tx; j < rn; j += 32) {
                double s = 0.0;
#pragma unroll
                for (int t = 0; t < 8; ++t) s += red[t][j];
                z[i + j * ldz] = s;
            }
        }
        __syncthreads();
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

__global__ void gaussian_transposed_kernel(double* __restrict__ out, int64_t rows, int64_t cols, uint64_t key) {
    const int64_t n = rows * cols;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = t / cols, j = t % cols;
        out[t] = normal_at_key(key, static_cast<uint64_t>(j * rows + c));
    }
}

template <typename T>
__global__ void gaussian_packed_kernel(T* __restrict__ out, int64_t rows, int cols, int stride, uint64_t key) {
    const int64_t n = rows * stride;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t c = t / stride;
        const int j = static_cast<int>(t % stride);
        out[t] = j < cols ? static_cast<T>(normal_at_key(key, static_cast<uint64_t>(j * rows + c))) : T(0);
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
    pack_factor_kernel<T><<<grid_for(rows * stride), 256, 0, s>>>(u, ld, rows, cols, stride, up);
    TK_LAUNCH_CHECK();
}

template <typename T>
void launch_sketch(const T* x, int64_t B, int64_t I, int64_t A, const double* omega_t, int rn, double* z,
                   int64_t ldz, cudaStream_t s) {
    require(rn >= 1 && rn <= kMaxRank, "sketch: r_tilde must be in [1, 64]");
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(I, 148 * 8));
    sketch_kernel<T><<<grid, 256, 0, s>>>(x, B, I, A, omega_t, rn, z, ldz);
    TK_LAUNCH_CHECK();
}

void launch_gaussian_colmajor(double* out, int64_t rows, int64_t cols, uint64_t key, cudaStream_t s) {
    const uint64_t n = uint64_t(rows) * uint64_t(cols);
    gaussian_colmajor_kernel<<<grid_for(static_cast<int64_t>((n + 1) / 2)), 256, 0, s>>>(out, n, key);
    TK_LAUNCH_CHECK();
}

void launch_gaussian_transposed(double* out, int64_t rows, int64_t cols, uint64_t key, cudaStream_t s) {
    gaussian_transposed_kernel<<<grid_for(rows * cols), 256, 0, s>>>(out, rows, cols, key);
    TK_LAUNCH_CHECK();
}

template <typename T>
void launch_gaussian_packed(T* out, int64_t rows, int cols, uint64_t key, cudaStream_t s) {
    const int stride = pack_stride(cols);
    gaussian_packed_kernel<T><<<grid_for(rows * stride), 256, 0, s>>>(out, rows, cols, stride, key);
    TK_LAUNCH_CHECK();
}
template void launch_gaussian_packed<float>(float*, int64_t, int, uint64_t, cudaStream_t);
template void launch_gaussian_packed<double>(double*, int64_t, int, uint64_t, cudaStream_t);

template <typename S, typename D>
void launch_cast(const S* in, D* out, int64_t n, cudaStream_t s) {
    cast_kernel<S, D><<<grid_for(n), 256, 0, s>>>(in, out, n);
    TK_LAUNCH_CHECK();
}

template void launch_ttm<float>(const float*, const float*, float*, int64_t, int64_t, int64_t, int, cudaStream_t, int*,
                                float*, int64_t);
template void launch_ttm<double>(const double*, const double*, double*, int64_t, int64_t, int64_t, int, cudaStream_t,
                                 int*, double*, int64_t);
template void launch_pack_factor<float>(const double*, int64_t, int64_t, int, float*, cudaStream_t);
template void launch_pack_factor<double>(const double*, int64_t, int64_t, int, double*, cudaStream_t);
template void launch_sketch<float>(const float*, int64_t, int64_t, int64_t, const double*, int, double*, int64_t,
                                   cudaStream_t);
template void launch_sketch<double>(const double*, int64_t, int64_t, int64_t, const double*, int, double*, int64_t,
                                    cudaStream_t);
template void launch_cast<float, double>(const float*, double*, int64_t, cudaStream_t);
template void launch_cast<double, float>(const double*, float*, int64_t, cudaStream_t);
template void launch_cast<double, double>(const double*, double*, int64_t, cudaStream_t);
template void launch_cast<float, float>(const float*, float*, int64_t, cudaStream_t);

}  // namespace tkb
