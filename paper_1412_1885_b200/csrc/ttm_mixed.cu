// ttm_mixed.cu — the Y-streaming first stage in fp64 arithmetic over fp32 data (the
// decomposition's precision = fp64 mode, tk_tucker_opts.precision): out (fp64) = in (fp32,
// exact in fp64) x_mode U (fp64), i.e. the reference's ttm (tensor.hpp:151-176) evaluated in
// the reference's own precision on the fp32 tensor, without a 2x-sized fp64 copy of Y.
// Same structure as ttm_mmajor_kernel: a producer lane streams BM x 16 column tiles of the
// (P, K, Q) view (bulk async copies into a 4-deep mbarrier ring), 8 consumer warps hold TM
// rows x R fp64 accumulators each and run DFMAs against the resident factor rows.
#include <algorithm>

#include "kernels.cuh"

namespace tkb {

namespace {

constexpr int kMxConsumers = 256;
constexpr int kMxBK = 16;
constexpr int kMxStages = 4;

template <int R>
struct MixedCfg {
    static constexpr int R4 = (R + 3) / 4 * 4;
    static constexpr int TM = R <= 24 ? 2 : 1;  // rows per thread (fp64 accumulators <= ~100 registers)
    static constexpr int BM = kMxConsumers * TM;
    static constexpr size_t smem = size_t(kMxStages) * kMxBK * (BM * sizeof(float) + R4 * sizeof(double)) +
                                   2 * kMxStages * sizeof(uint64_t);
};

// out[p + r P + q P cols] = sum_k double(in[p + k P + q P K]) * up[k R4 + r]
template <int R>
__global__ void __launch_bounds__(kMxConsumers + 32, 1)
    ttm_mixed_kernel(const float* __restrict__ in, const double* __restrict__ up, double* __restrict__ out, int64_t P,
                     int64_t K, int cols, int64_t tiles_p, int64_t ntiles) {
    using Cfg = MixedCfg<R>;
    constexpr int R4 = Cfg::R4, TM = Cfg::TM, BM = Cfg::BM;
    extern __shared__ __align__(128) unsigned char mx_smem[];
    float* sY = reinterpret_cast<float*>(mx_smem);                                   // [stages][BK][BM]
    double* sU = reinterpret_cast<double*>(sY + kMxStages * kMxBK * BM);               // [stages][BK][R4]
    uint64_t* full = reinterpret_cast<uint64_t*>(sU + kMxStages * kMxBK * R4);
    uint64_t* empty = full + kMxStages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = static_cast<int>((K + kMxBK - 1) / kMxBK);
    if (tid == 0) {
        for (int s = 0; s < kMxStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kMxConsumers / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == kMxConsumers / 32) {  // producer: persistent over tiles
        if (lane == 0) {
            uint32_t g = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t q = t / tiles_p, p0 = (t % tiles_p) * BM;
                const int rows = static_cast<int>(lmin(BM, P - p0));
                const float* base = in + q * P * K + p0;
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    const int s = static_cast<int>(g % kMxStages);
                    mbar_wait(&empty[s], ((g / kMxStages) & 1) ^ 1);
                    const int64_t k0 = int64_t(kc) * kMxBK;
                    const int kn = static_cast<int>(lmin(kMxBK, K - k0));
                    const uint32_t ybytes = uint32_t(rows) * sizeof(float);
                    mbar_arrive_expect_tx(&full[s], ybytes * kn + uint32_t(kn) * R4 * sizeof(double));
                    for (int kk = 0; kk < kn; ++kk)
                        bulk_g2s(sY + (s * kMxBK + kk) * BM, base + (k0 + kk) * P, ybytes, &full[s]);
                    bulk_g2s(sU + s * kMxBK * R4, up + k0 * R4, uint32_t(kn) * R4 * sizeof(double), &full[s]);
                }
            }
        }
        return;
    }
    uint32_t g = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t q = t / tiles_p, p0 = (t % tiles_p) * BM;
        const int rows = static_cast<int>(lmin(BM, P - p0));
        double acc[TM][R];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int r = 0; r < R; ++r) acc[i][r] = 0.0;
        for (int kc = 0; kc < nk; ++kc, ++g) {
            const int s = static_cast<int>(g % kMxStages);
            mbar_wait(&full[s], (g / kMxStages) & 1);
            const int kn = static_cast<int>(lmin(kMxBK, K - int64_t(kc) * kMxBK));
            const float* ys = sY + s * kMxBK * BM + tid * TM;
            const double* us = sU + s * kMxBK * R4;
            for (int kk = 0; kk < kn; ++kk) {
                double y[TM];
                if constexpr (TM == 2) {
                    const float2 v = *reinterpret_cast<const float2*>(ys + kk * BM);
                    y[0] = v.x, y[1] = v.y;
                } else {
                    y[0] = ys[kk * BM];
                }
                const double* ur = us + kk * R4;
#pragma unroll
                for (int r = 0; r < R; r += 2) {
                    const double2 u = *reinterpret_cast<const double2*>(ur + r);
#pragma unroll
                    for (int i = 0; i < TM; ++i) {
                        acc[i][r] = fma(y[i], u.x, acc[i][r]);
                        if (r + 1 < R) acc[i][r + 1] = fma(y[i], u.y, acc[i][r + 1]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (tid * TM < rows) {
            double* o = out + q * P * cols + p0 + tid * TM;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r < cols)
#pragma unroll
                    for (int i = 0; i < TM; ++i)
                        if (tid * TM + i < rows) o[int64_t(r) * P + i] = acc[i][r];
        }
    }
}

template <int R>
void launch_mixed(const float* in, const double* up, double* out, int64_t P, int64_t K, int64_t Q, int cols,
                  cudaStream_t s) {
    using Cfg = MixedCfg<R>;
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(ttm_mixed_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(Cfg::smem)));
        attr = true;
    }
    const int64_t tiles_p = (P + Cfg::BM - 1) / Cfg::BM;
    const int64_t ntiles = tiles_p * Q;
    const int64_t grid = std::min<int64_t>(ntiles, 148);
    TK_MAXSMEM((ttm_mixed_kernel<R>));
    ttm_mixed_kernel<R><<<static_cast<unsigned>(grid), kMxConsumers + 32, Cfg::smem, s>>>(in, up, out, P, K, cols,
                                                                                          tiles_p, ntiles);
    TK_LAUNCH_CHECK();
}

}  // namespace

bool mixed_ttm_supported(const float* in, int64_t P) {
    return P % 4 == 0 && P >= 64 && reinterpret_cast<uintptr_t>(in) % 16 == 0;
}

// up: the factor packed k-major with stride pack_stride(cols) (launch_pack_factor<double>)
void launch_ttm_mixed(const float* in, const double* up, double* out, int64_t P, int64_t K, int64_t Q, int cols,
                      cudaStream_t s) {
    require(cols >= 1 && cols <= kMaxRank, "ttm: factor column count must be in [1, 64]");
    require(mixed_ttm_supported(in, P), "ttm: the fp64 mode's first stage needs a leading extent % 4 == 0");
    switch (pack_stride(cols)) {
        case 4: return launch_mixed<4>(in, up, out, P, K, Q, cols, s);
        case 8: return launch_mixed<8>(in, up, out, P, K, Q, cols, s);
        case 12: return launch_mixed<12>(in, up, out, P, K, Q, cols, s);
        case 16: return launch_mixed<16>(in, up, out, P, K, Q, cols, s);
        case 20: return launch_mixed<20>(in, up, out, P, K, Q, cols, s);
        case 24: return launch_mixed<24>(in, up, out, P, K, Q, cols, s);
        case 28: return launch_mixed<28>(in, up, out, P, K, Q, cols, s);
        case 32: return launch_mixed<32>(in, up, out, P, K, Q, cols, s);
        case 36: return launch_mixed<36>(in, up, out, P, K, Q, cols, s);
        case 40: return launch_mixed<40>(in, up, out, P, K, Q, cols, s);
        case 44: return launch_mixed<44>(in, up, out, P, K, Q, cols, s);
        case 48: return launch_mixed<48>(in, up, out, P, K, Q, cols, s);
        case 52: return launch_mixed<52>(in, up, out, P, K, Q, cols, s);
        case 56: return launch_mixed<56>(in, up, out, P, K, Q, cols, s);
        case 60: return launch_mixed<60>(in, up, out, P, K, Q, cols, s);
        default: return launch_mixed<64>(in, up, out, P, K, Q, cols, s);
    }
}

}  // namespace tkb
