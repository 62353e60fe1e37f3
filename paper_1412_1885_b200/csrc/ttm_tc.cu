// ttm_tc.cu — the Y-streaming TTM on the 5th-generation tensor cores (tcgen05, sm_100a).
//
// Same contraction as ttm_mmajor_kernel (out[p, r, q] = sum_k Y[p, k, q] U[k, r], the
// first stage of every X_n = Y x_{p != n} U_p^T, tensor.hpp:151-192), but the FFMA loop is
// replaced by tf32 UMMAs in an fp32-accurate 3-pass split (plain TF32 flips
// the sign rule; 3xTF32 keeps ~2^-21 relative error per product):
//     y u ~= y_hi u_hi + y_hi u_lo + y_lo u_hi,   x_hi = rna_tf32(x), x_lo = x - x_hi (exact)
// Warp roles (one 512-row tile of Y per CTA, K streamed in 16-column stages):
//   warp 8      producer: TMA tensor loads (BOXR-row x 16-k boxes of the (P, K, Q) view,
//               zero-filled out of bounds) + a bulk copy of the packed [U_hi | U_lo] stage
//               into a 4-deep shared-memory ring (mbarrier complete_tx)
//   warps 0-7   converters: LDS.128 of 4 rows per thread, split y into (hi, lo) and
//               tcgen05.st them as the A operands in TMEM (row 4L+j of the tile goes to
//               TMEM lane L of M-tile j; warps w and w+4 share lane quarter w and split the
//               16 k of a stage), then the epilogue (warps 0-3: tcgen05.ld, D_hi + D_lo)
//   warp 9      TMEM allocator + single-thread MMA issuer:
//               D_j[0:2NH] += A_hi_j [U_hi | U_lo]   (N = 2NH)
//               D_j[0:NH]  += A_lo_j  U_hi           (N = NH)
// Accumulators stay in TMEM for the whole K loop; Y is read from HBM exactly once.
#include <cuda.h>

#include <cstdlib>
#include <stdexcept>

namespace {
// The driver entry point is resolved through the runtime (no link-time libcuda dependency,
// so the library loads on hosts without a driver and fails only when a kernel is launched).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        return (e == cudaSuccess && q == cudaDriverEntryPointSuccess) ? reinterpret_cast<EncodeTiledFn>(p) : nullptr;
    }();
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
    return fn;
}
}  // namespace

#include <algorithm>

#include "kernels.cuh"

namespace tkb {

namespace {

constexpr int kTcConv = 8;                      // converter warps: 2 per TMEM lane quarter (k halves)
constexpr int kTcThreads = (kTcConv + 2) * 32;  // + producer warp + MMA warp
constexpr int kTcBK = 16;                       // K per pipeline stage (2 MMA k-steps of 8)
constexpr int kTcStages = 4;
// 3xTF32: y_hi u_hi -> main accumulators, y_hi u_lo + y_lo u_hi -> cross accumulator (the
// fourth product y_lo u_lo, 2^-22 relative, is dropped).

template <int NH, int MT_ = (NH <= 32 ? 4 : 2), int OCC_ = 1>
struct TcCfg {
    static constexpr int OCC = OCC_;            // CTAs per SM (TMEM and smem split between them)
    static constexpr int TMEM = 512 / OCC_;
    static constexpr int MT = MT_;  // 128-row M tiles per CTA
    static constexpr int BM = 128 * MT;
    static constexpr int BOXR = BM < 256 ? BM : 256;  // rows per TMA box
    static constexpr int BBYTES = 64 * NH;       // one k-step of [U_hi | U_lo]: 2NH rows x 8 tf32
    static constexpr int STAGE_Y = kTcBK * BM * 4;
    static constexpr int STAGE_B = 2 * BBYTES;
    static constexpr int D_COLS = MT * 2 * NH;   // one accumulator set: per tile [main | cross]
    static constexpr int A_COLS = MT * 32;       // per A stage and tile: 16 hi + 16 lo columns
    static constexpr int XBASE = D_COLS + 2 * A_COLS;  // accumulator sets 1.. (D_COLS each)
    // The fp32 accumulation inside the tensor core truncates, so its error grows with the
    // number of MMAs accumulated into one D: k-block kc accumulates into set kc % S, and the
    // sets are summed in round-to-nearest fp32 in the epilogue.
    static constexpr int S_RAW = 1 + (TMEM - XBASE) / D_COLS;
    static constexpr int S = S_RAW > 4 ? 4 : S_RAW;
    static_assert(XBASE <= TMEM, "TMEM budget");
    // pipeline depth: ~128 KB of Y in flight per SM whatever the tile height
    static constexpr int STAGES_RAW = (128 * 1024) / STAGE_Y / OCC_;
    // at most 8 stages and what fits OCC CTAs into the SM's shared memory
    static constexpr int STAGES_FIT = (220 * 1024 / OCC_ - 1024) / (STAGE_Y + STAGE_B);
    static constexpr int STAGES_CAP = STAGES_FIT < 8 ? STAGES_FIT : 8;
    static constexpr int STAGES = STAGES_RAW < kTcStages ? kTcStages : (STAGES_RAW > STAGES_CAP ? STAGES_CAP : STAGES_RAW);
    static constexpr size_t smem = size_t(STAGES) * (STAGE_Y + STAGE_B) + 256 + 128;
};

__device__ __forceinline__ uint32_t f2tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
    return r;
}

// round-to-nearest (ties away) to tf32 on the magnitude bits; the residual x - hi is exact
// in fp32 and is handed to the MMA as is (the tensor core reads its top 19 bits; rounding it
// first changed nothing measurable and costs converter issue slots)
__device__ __forceinline__ uint32_t tf32_hi_bits(float x) { return (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u; }

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr)
        : "memory");
}

// UMMA shared-memory descriptor: K-major, no swizzle (core matrices of 8 rows x 16 B),
// LBO = 128 B between the two 16-B K chunks of a k-step, SBO = 256 B between 8-row groups.
__device__ __forceinline__ uint64_t bdesc(const void* smem) {
    const uint64_t a = smem_u32(smem);
    return ((a >> 4) & 0x3FFFull) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
}

// Instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = n.
__device__ __forceinline__ uint32_t idesc_tf32(int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(0u), "r"(0u), "r"(0u), "r"(0u)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

// Columns rc..rc+15 of tile j: sum over the accumulator sets of (main + cross), in
// round-to-nearest fp32 (`used` = sets actually written: min(k-blocks, S)).
template <class C>
__device__ __forceinline__ void drain16(uint32_t tl, int j, int rc, int used, float (&v)[16]) {
    constexpr int NH = C::D_COLS / (2 * C::MT);
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = 0.f;
    for (int sm = 0; sm < used; ++sm) {
        const uint32_t base = tl + uint32_t((sm == 0 ? 0 : C::XBASE + (sm - 1) * C::D_COLS) + j * 2 * NH + rc);
        uint32_t uh[16], ul[16];
        tmem_ld16(base, uh);
        tmem_ld16(base + NH, ul);
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] += __uint_as_float(uh[e]) + __uint_as_float(ul[e]);
    }
}

// KM = false: the contracted mode is not the fastest (P > 1): Y viewed as (P, K, Q), tiles of
//   BM consecutive p for one q, TMA boxes of 256 p x 16 k, out[p + r P + q P cols].
// KM = true: the contracted mode is mode 0 (P == 1): Y viewed as Q rows of K contiguous
//   values, tiles of BM rows, TMA boxes of BOXR rows x 16 k (64 B, 64B-swizzled so the
//   converters' 16-B row reads are bank-conflict free), out[r + q cols] written through a
//   shared-memory transpose (coalesced rows of the output).
template <int NH, int MT_, bool KM, int OCC = 1>
__global__ void __launch_bounds__(kTcThreads, OCC)
    ttm_tc_kernel(const __grid_constant__ CUtensorMap ymap, const uint8_t* __restrict__ bpk, float* __restrict__ out,
                  int64_t P, int64_t K, int cols, int64_t tiles_p, int tout, int64_t ntiles) {
    using C = TcCfg<NH, MT_, OCC>;
    constexpr int MT = C::MT, BM = C::BM;
    extern __shared__ __align__(1024) uint8_t tsm[];
    uint8_t* sY = tsm;  // [stages][BM/BOXR boxes][kTcBK][BOXR] fp32
    uint8_t* sB = tsm + size_t(C::STAGES) * C::STAGE_Y;           // [stages][2][2NH x 8] tf32 core matrices
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(C::STAGES) * C::STAGE_B);
    uint64_t* full = bars;                   // [stages]  producer -> (converters, MMA)
    uint64_t* empty = bars + C::STAGES;      // [stages]  converters (4) + MMA commit (1) -> producer
    uint64_t* afull = bars + 2 * C::STAGES;  // [2]       converters -> MMA
    uint64_t* aempty = afull + 2;            // [2]       MMA commit -> converters
    uint64_t* dfull = aempty + 2;            // [1]       MMA commit -> epilogue
    uint64_t* dempty = dfull + 1;            // [1]       epilogue warps (D drained) -> MMA of the next tile
    uint32_t* tbase_sm = reinterpret_cast<uint32_t*>(dempty + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // split-K (gridDim.y > 1): this CTA takes k-blocks [kb0, kb0 + nk) and writes its partial
    // to out + blockIdx.y * (P * cols * Q); the caller sums the partials in split order
    const int nk_all = static_cast<int>((K + kTcBK - 1) / kTcBK);
    const int nk_per = (nk_all + static_cast<int>(gridDim.y) - 1) / static_cast<int>(gridDim.y);
    const int kb0 = static_cast<int>(blockIdx.y) * nk_per;
    const int nk = nk_per < nk_all - kb0 ? nk_per : nk_all - kb0;
    out += int64_t(blockIdx.y) * P * cols * (ntiles / tiles_p);

    if (tid == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kTcConv + 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&afull[a], kTcConv);
            mbar_init(&aempty[a], 1);
        }
        mbar_init(dfull, 1);
        mbar_init(dempty, kTcConv / 2);
        mbar_fence_init();
    }
    if (warp == kTcConv + 1) {  // TMEM allocation (whole warp)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tbase_sm)),
                     "r"(C::TMEM));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tbase_sm;

    // Tiles blockIdx.x, blockIdx.x + gridDim.x, ...: a persistent launch (gridDim.x < ntiles)
    // keeps the ring streaming across tile boundaries — the producer loads the next tile while
    // this one is multiplied and drained; the MMA of the next tile waits only for the drain of
    // D (dempty). Stage / A-buffer phases run on a per-CTA counter g over all tiles.
    if (warp == kTcConv) {
        // ===== producer =====
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];\n" ::"l"(&ymap) : "memory");
            uint32_t g = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                const int64_t q = t / tiles_p;
                const int64_t p0 = (t % tiles_p) * BM;
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    const int s = static_cast<int>(g % C::STAGES);
                    mbar_wait(&empty[s], ((g / C::STAGES) & 1) ^ 1);
                    mbar_arrive_expect_tx(&full[s], C::STAGE_Y + C::STAGE_B);
                    uint8_t* dy = sY + size_t(s) * C::STAGE_Y;
                    if constexpr (KM) {
#pragma unroll
                        for (int b = 0; b < BM / C::BOXR; ++b)
                            tma_load_2d(dy + b * (C::BOXR * kTcBK * 4), &ymap, (kb0 + kc) * kTcBK,
                                        static_cast<int>(p0 + C::BOXR * b), &full[s]);
                    } else {
#pragma unroll
                        for (int b = 0; b < BM / C::BOXR; ++b)
                            tma_load_3d(dy + b * (kTcBK * C::BOXR * 4), &ymap, static_cast<int>(p0 + C::BOXR * b),
                                        (kb0 + kc) * kTcBK, static_cast<int>(q), &full[s]);
                    }
                    bulk_g2s(sB + size_t(s) * C::STAGE_B, bpk + size_t(kb0 + kc) * C::STAGE_B, C::STAGE_B, &full[s]);
                }
            }
        }
    } else if (warp == kTcConv + 1) {
        // ===== MMA issuer =====
        if (lane == 0) {
            const uint32_t id_full = idesc_tf32(2 * NH), id_hi = idesc_tf32(NH);
            uint32_t g = 0, it = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
                if (it > 0) {  // the previous tile's D must be drained before it is overwritten
                    mbar_wait(dempty, (it - 1) & 1);
                    fence_after();
                }
                for (int kc = 0; kc < nk; ++kc, ++g) {
                    const int s = static_cast<int>(g % C::STAGES), a = static_cast<int>(g & 1);
                    mbar_wait(&full[s], (g / C::STAGES) & 1);
                    mbar_wait(&afull[a], (g >> 1) & 1);
                    fence_after();
                    const uint8_t* bs = sB + size_t(s) * C::STAGE_B;
#pragma unroll
                    for (int j = 0; j < MT; ++j) {
                        const int sm = kc % C::S;
                        // set sm, tile j: [main | cross]; y_hi [u_hi | u_lo] fills both halves,
                        // y_lo u_hi adds into the cross half (main keeps only y_hi u_hi)
                        const uint32_t d = tmem + uint32_t((sm == 0 ? 0 : C::XBASE + (sm - 1) * C::D_COLS) + j * 2 * NH);
                        const uint32_t ahi = tmem + uint32_t(C::D_COLS + a * C::A_COLS + j * 32);
#pragma unroll
                        for (int ks = 0; ks < 2; ++ks) {
                            const uint64_t b = bdesc(bs + ks * C::BBYTES);
                            mma_tf32_ts(d, ahi + ks * 8, b, id_full, (kc >= C::S || ks > 0) ? 1u : 0u);
                            mma_tf32_ts(d + NH, ahi + 16 + ks * 8, b, id_hi, 1u);
                        }
                    }
                    mma_commit(&aempty[a]);
                    mma_commit(&empty[s]);
                }
                mma_commit(dfull);
            }
        }
    } else {
        // ===== converters (warps 0-7): Y tile -> (hi, lo) tf32 A operands in TMEM =====
        const int quarter = warp & 3, khalf = warp >> 2;
        const int L = quarter * 32 + lane;                    // TMEM lane of this thread
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        uint32_t g = 0, it = 0;
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int64_t q = t / tiles_p;
            const int64_t p0 = (t % tiles_p) * BM;
            const int rows = static_cast<int>(lmin(BM, P - p0));
            for (int kc = 0; kc < nk; ++kc, ++g) {
                const int s = static_cast<int>(g % C::STAGES), a = static_cast<int>(g & 1);
                mbar_wait(&full[s], (g / C::STAGES) & 1);
                uint32_t hi[MT][8], lo[MT][8];
                // rows MT*L .. MT*L+MT-1 of the tile sit in box (MT*L)/BOXR at row (MT*L)%BOXR
                const float* ys = reinterpret_cast<const float*>(sY + size_t(s) * C::STAGE_Y) +
                                  ((MT * L) / C::BOXR) * (kTcBK * C::BOXR) + (MT * L) % C::BOXR + khalf * 8 * C::BOXR;
                if constexpr (KM) {
                    // row j*128 + L of the tile: 8 k values = logical 16-B chunks 2*khalf, 2*khalf+1
                    const uint8_t* stage = sY + size_t(s) * C::STAGE_Y;
#pragma unroll
                    for (int j = 0; j < MT; ++j) {
                        const int row = j * 128 + L;
                        const int rr = row % C::BOXR;
                        const uint8_t* rb = stage + (row / C::BOXR) * (C::BOXR * kTcBK * 4) + rr * 64;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int phys = (2 * khalf + h) ^ ((rr >> 1) & 3);
                            const float4 v = *reinterpret_cast<const float4*>(rb + phys * 16);
                            const float y4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                            for (int e = 0; e < 4; ++e) {
                                const uint32_t hb = tf32_hi_bits(y4[e]);
                                hi[j][h * 4 + e] = hb;
                                lo[j][h * 4 + e] = __float_as_uint(y4[e] - __uint_as_float(hb));
                            }
                        }
                    }
                } else {
                    auto split = [&](int kk, bool live) {
                        float y[MT];
                        if constexpr (MT == 4) {
                            const float4 v = *reinterpret_cast<const float4*>(ys + kk * C::BOXR);
                            y[0] = v.x, y[1] = v.y, y[2] = v.z, y[3] = v.w;
                        } else if constexpr (MT == 2) {
                            const float2 v = *reinterpret_cast<const float2*>(ys + kk * C::BOXR);
                            y[0] = v.x, y[1] = v.y;
                        } else {
                            y[0] = ys[kk * C::BOXR];
                        }
#pragma unroll
                        for (int j = 0; j < MT; ++j) {
                            const float x = live ? y[j] : 0.f;
                            const uint32_t h = tf32_hi_bits(x);
                            hi[j][kk] = h;
                            lo[j][kk] = __float_as_uint(x - __uint_as_float(h));
                        }
                    };
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk) split(kk, true);  // the K tail is zero-filled by the TMA
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);  // Y stage consumed (B: the MMA commit)
                mbar_wait(&aempty[a], ((g >> 1) & 1) ^ 1);
                fence_after();
#pragma unroll
                for (int j = 0; j < MT; ++j) {
                    const uint32_t ta = tmem + lane_off + uint32_t(C::D_COLS + a * C::A_COLS + j * 32 + khalf * 8);
                    tmem_st8(ta, hi[j]);
                    tmem_st8(ta + 16, lo[j]);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&afull[a]);
            }
            if (khalf == 1) continue;  // the epilogue runs on warps 0-3 (one per lane quarter)
            // ===== epilogue: D = D[:, 0:NH] + D[:, NH:2NH], rows MT*L + j =====
            mbar_wait(dfull, it & 1);
            fence_after();
            if (KM && !tout) {
                // (never persistent: the staging reuses the Y ring.) D tile j, TMEM lane L = row
                // j*128 + L: stage [row][cols] in the (drained) Y buffers, then copy the
                // contiguous out[p0*cols ...] block with coalesced stores
                float* stg = reinterpret_cast<float*>(sY);
#pragma unroll
                for (int rc = 0; rc < NH; rc += 16) {
#pragma unroll
                    for (int j = 0; j < MT; ++j) {
                        float v[16];
                        drain16<C>(tmem + lane_off, j, rc, min(nk, C::S), v);
                        float* srow = stg + (j * 128 + L) * cols;
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (rc + e < cols) srow[rc + e] = v[e];
                    }
                }
                asm volatile("bar.sync 1, 128;\n" ::: "memory");
                const int64_t n = int64_t(rows) * cols;
                float* o = out + p0 * cols;
                for (int64_t e = tid; e < n; e += 128) o[e] = stg[e];
            } else {
                float* o = out + q * P * cols + p0 + MT * L;
                const bool live = MT * L < rows;
#pragma unroll
                for (int rc = 0; rc < NH; rc += 16) {
                    float acc[MT][16];
#pragma unroll
                    for (int j = 0; j < MT; ++j) drain16<C>(tmem + lane_off, j, rc, min(nk, C::S), acc[j]);
                    if (live) {
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const int r = rc + e;
                            if (r < cols) {
                                if constexpr (MT == 4) {
                                    *reinterpret_cast<float4*>(o + int64_t(r) * P) =
                                        make_float4(acc[0][e], acc[1][e], acc[2][e], acc[3][e]);
                                } else if constexpr (MT == 2) {
                                    *reinterpret_cast<float2*>(o + int64_t(r) * P) = make_float2(acc[0][e], acc[1][e]);
                                } else {
                                    o[int64_t(r) * P] = acc[0][e];
                                }
                            }
                        }
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dempty);  // D drained: the next tile's MMAs may overwrite it
        }
    }
    fence_before();
    __syncthreads();
    if (warp == kTcConv + 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(C::TMEM));
    }
}

// [U_hi | U_lo] of a column-major fp64 factor (rows x cols, ld), tf32 in the UMMA K-major
// no-swizzle core-matrix layout, one 64*NH-byte block per k-step of 8 rows of U.
template <int NH>
__global__ void pack_umma_kernel(const double* __restrict__ u, int64_t ld, int64_t rows, int cols, int64_t ksteps,
                                 uint32_t* __restrict__ out) {
    const int64_t n_el = ksteps * 2 * NH * 8;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n_el; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = t / (2 * NH * 8);
        const int rem = static_cast<int>(t % (2 * NH * 8));
        const int n = rem / 8, kk = rem % 8;
        const int64_t k = g * 8 + kk;
        const int r = n < NH ? n : n - NH;
        const float uf = (k < rows && r < cols) ? static_cast<float>(u[k + int64_t(r) * ld]) : 0.f;
        const uint32_t h = f2tf32(uf);
        const uint32_t v = n < NH ? h : f2tf32(uf - __uint_as_float(h));
        const int64_t byte = g * (64 * NH) + (n / 8) * 256 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4;
        out[byte / 4] = v;
    }
}

template <int NH, int MT, bool KM, int OCC = 1>
void launch_tc(const float* in, const uint8_t* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
               cudaStream_t s, bool tout = false, int splits = 1) {
    using C = TcCfg<NH, MT, OCC>;
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(ttm_tc_kernel<NH, MT, KM, OCC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(C::smem)));
        attr = true;
    }
    require(K < (int64_t(1) << 31) && Q < (int64_t(1) << 31) && P < (int64_t(1) << 31), "ttm: extent too large for TMA");
    CUtensorMap map;
    CUresult r;
    int64_t tiles_p, grid;
    if constexpr (KM) {  // rows q of K contiguous values
        tiles_p = (Q + C::BM - 1) / C::BM;
        grid = tiles_p;
        const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(Q)};
        const cuuint64_t strides[1] = {cuuint64_t(K) * 4};
        const cuuint32_t box[2] = {kTcBK, C::BOXR};
        const cuuint32_t estr[2] = {1, 1};
        r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(in), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        P = Q;  // the kernel's row extent
    } else {
        tiles_p = (P + C::BM - 1) / C::BM;
        grid = tiles_p * Q;
        const cuuint64_t dims[3] = {cuuint64_t(P), cuuint64_t(K), cuuint64_t(Q)};
        const cuuint64_t strides[2] = {cuuint64_t(P) * 4, cuuint64_t(P) * cuuint64_t(K) * 4};
        const cuuint32_t box[3] = {C::BOXR, kTcBK, 1};
        const cuuint32_t estr[3] = {1, 1, 1};
        r = encode_tiled()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    require(grid < (int64_t(1) << 31), "ttm: grid too large");
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    // Persistent launch (OCC CTAs per SM looping over tiles) for the streaming shapes with many
    // tiles; the K-major second stage (transpose staged through the Y ring) stays one tile per CTA.
    static const int persist = [] {
        const char* e = std::getenv("TENKIT_TC_PERSIST");
        return e ? std::atoi(e) : 1;
    }();
    const int64_t ntiles = grid;
    const int64_t slots = int64_t(148) * OCC;
    if (persist && !(KM && !tout) && splits == 1 && grid > 2 * slots) grid = slots;
    TK_MAXSMEM((ttm_tc_kernel<NH, MT, KM, OCC>));
    ttm_tc_kernel<NH, MT, KM, OCC><<<dim3(static_cast<unsigned>(grid), static_cast<unsigned>(splits)), kTcThreads,
                                     C::smem, s>>>(map, bpk, out, P, K, cols, tiles_p, tout ? 1 : 0, ntiles);
    TK_LAUNCH_CHECK();
}

inline int tc_nh(int cols) { return cols <= 16 ? 16 : cols <= 32 ? 32 : cols <= 48 ? 48 : 64; }

}  // namespace

int64_t umma_pack_bytes(int64_t rows, int cols) {
    const int64_t ksteps = (rows + kTcBK - 1) / kTcBK * 2;
    return ksteps * 64 * tc_nh(cols);
}

void launch_pack_umma(const double* u, int64_t ld, int64_t rows, int cols, void* out, cudaStream_t s) {
    require(cols >= 1 && cols <= kMaxRank, "ttm: factor column count must be in [1, 64]");
    const int64_t ksteps = (rows + kTcBK - 1) / kTcBK * 2;
    const int nh = tc_nh(cols);
    const int64_t n = ksteps * 2 * nh * 8;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
    uint32_t* o = static_cast<uint32_t*>(out);
    switch (nh) {
        case 16: TK_MAXSMEM((pack_umma_kernel<16>)); pack_umma_kernel<16><<<grid, 256, 0, s>>>(u, ld, rows, cols, ksteps, o); break;
        case 32: TK_MAXSMEM((pack_umma_kernel<32>)); pack_umma_kernel<32><<<grid, 256, 0, s>>>(u, ld, rows, cols, ksteps, o); break;
        case 48: TK_MAXSMEM((pack_umma_kernel<48>)); pack_umma_kernel<48><<<grid, 256, 0, s>>>(u, ld, rows, cols, ksteps, o); break;
        default: TK_MAXSMEM((pack_umma_kernel<64>)); pack_umma_kernel<64><<<grid, 256, 0, s>>>(u, ld, rows, cols, ksteps, o); break;
    }
    TK_LAUNCH_CHECK();
}

// Y-streaming passes: two CTAs per SM, each with 2 x 128-row tiles, 256 TMEM columns and a
// 4-stage ring (one CTA's prologue, pipeline fill and epilogue overlap the other's stream:
// 6.1 TB/s vs 5.4 TB/s for one 512-row CTA per SM at cfg 2). TMEM then holds one accumulator
// set (the main accumulator takes one MMA per k-step). Short contractions that cannot fill
// the GPU with such tiles (K-major second stages) use 128-row tiles, 2 CTAs per SM and 3
// accumulator sets.
inline bool km_wide(int64_t Q) { return (Q + 255) / 256 >= 4 * 148; }
constexpr int kMmt = 2;
constexpr int kOcc = 2;

inline int64_t mm_tiles(int64_t P, int64_t Q, int cols) {
    const int bm = tc_nh(cols) <= 32 ? 128 * kMmt : 128;
    return (P + bm - 1) / bm * Q;
}

// Split-K factor for an M-major contraction whose row tiles alone cannot fill 2 waves of 2
// CTAs per SM: >= 8 k-blocks (128 k) per split, no empty split, partials fit `work_elems`.
inline int mm_splits(int64_t P, int64_t K, int64_t Q, int cols, int64_t work_elems) {
    const int64_t tiles = mm_tiles(P, Q, cols);
    if (tiles >= 2 * 2 * 148) return 1;
    const int64_t nk = (K + kTcBK - 1) / kTcBK;
    int64_t sp = std::min<int64_t>((2 * 2 * 148 + tiles - 1) / tiles, nk / 8);
    sp = std::min<int64_t>(sp, work_elems / std::max<int64_t>(1, P * cols * Q));
    if (sp < 2) return 1;
    const int64_t per = (nk + sp - 1) / sp;
    return static_cast<int>((nk + per - 1) / per);
}

bool tc_ttm_supported(const float* in, float* out, int64_t P, int64_t K, int64_t Q, int cols, int64_t work_elems) {
    if (reinterpret_cast<uintptr_t>(in) % 16 != 0 || reinterpret_cast<uintptr_t>(out) % 16 != 0) return false;
    // K-major: R~ <= 48 (NH = 48 keeps 2 accumulator sets in 256 TMEM columns at MT = 1)
    // (R~ <= 64: NH = 64 on one CTA per SM, 512 TMEM columns, 3 accumulator sets)
    if (P == 1) return K % 4 == 0 && K >= kTcBK && cols <= 64 && (Q + 127) / 128 >= 148;
    if (P % 4 != 0 || P < 256) return false;
    // tiles >= 2 waves of 2 CTAs per SM, or (with split-K partials) >= 1 wave
    const int64_t tiles = mm_tiles(P, Q, cols);
    return tiles >= 2 * 2 * 148 || tiles * mm_splits(P, K, Q, cols, work_elems) >= 2 * 148;
}

int launch_ttm_tc(const float* in, const void* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                  cudaStream_t s, bool accurate, bool tout, float* work, int64_t work_elems) {
    const uint8_t* b = static_cast<const uint8_t*>(bpk);
    if (P == 1) {
        const bool wide = km_wide(Q) && !accurate && !tout;  // narrow tiles: 3 accumulator sets
        if (tc_nh(cols) <= 16) wide ? launch_tc<16, 2, true, 2>(in, b, out, P, K, Q, cols, s, tout)
                                    : launch_tc<16, 1, true, 2>(in, b, out, P, K, Q, cols, s, tout);
        else if (tc_nh(cols) <= 32) wide ? launch_tc<32, 2, true, 2>(in, b, out, P, K, Q, cols, s, tout)
                                         : launch_tc<32, 1, true, 2>(in, b, out, P, K, Q, cols, s, tout);
        else if (tc_nh(cols) <= 48) launch_tc<48, 1, true, 2>(in, b, out, P, K, Q, cols, s, tout);
        else launch_tc<64, 1, true, 1>(in, b, out, P, K, Q, cols, s, tout);
        return 1;
    }
    static const int variant = [] {
        const char* e = std::getenv("TENKIT_TC_VARIANT");
        return e ? std::atoi(e) : 0;
    }();
    if (variant == 1) {  // A/B: one CTA per SM (the round-1 first version)
        if (tc_nh(cols) <= 16) launch_tc<16, 4, false>(in, b, out, P, K, Q, cols, s);
        else if (tc_nh(cols) <= 32) launch_tc<32, 4, false>(in, b, out, P, K, Q, cols, s);
        else if (tc_nh(cols) <= 48) launch_tc<48, 2, false>(in, b, out, P, K, Q, cols, s);
        else launch_tc<64, 2, false>(in, b, out, P, K, Q, cols, s);
        return 1;
    }
    const int sp = work ? mm_splits(P, K, Q, cols, work_elems) : 1;
    float* dst = sp > 1 ? work : out;
    switch (tc_nh(cols)) {
        case 16: launch_tc<16, kMmt, false, kOcc>(in, b, dst, P, K, Q, cols, s, false, sp); break;
        case 32: launch_tc<32, kMmt, false, kOcc>(in, b, dst, P, K, Q, cols, s, false, sp); break;
        // wider factors: one 128-row tile per CTA keeps two CTAs per SM inside 256 TMEM columns
        case 48: launch_tc<48, 1, false, kOcc>(in, b, dst, P, K, Q, cols, s, false, sp); break;
        default: launch_tc<64, 1, false, kOcc>(in, b, dst, P, K, Q, cols, s, false, sp); break;
    }
    if (sp > 1) launch_splitk_reduce<float>(work, out, P * cols * Q, sp, s);
    return sp > 1 ? 2 : 1;
}

}  // namespace tkb
