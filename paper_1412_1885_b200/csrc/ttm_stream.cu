// ttm_stream.cu — the Y-streaming pass (first stage of every X_n = Y x_{p != n} U_p^T and of
// the core, tensor.hpp:151-192) on the tcgen05 tensor cores, second design.
//
//   out[p, r, q] = sum_k Y[p, k, q] U[k, r]       (3xTF32: y u ~= y_hi u_hi + y_hi u_lo + y_lo u_hi)
//
// Differences from ttm_tc.cu (the first design, still used for the second stages):
// * y_hi is read by the MMA straight from the TMA-staged shared memory: the tensor core takes
//   the top 19 bits of an fp32 operand (y_hi = trunc_tf32(y)), so only y_lo = y - y_hi (exact)
//   is computed by the converter warps and stored to TMEM (half the TMEM stores, and the main
//   MMAs no longer wait for the converters). M-major tiles (contracted mode not the fastest)
//   are MN-major A operands (TMA boxes of 32 p x 16 k; MN-major tf32 takes only the 128B-span
//   swizzle with 32-B atoms), K-major tiles (mode 0) K-major A operands (16 k x rows, 64B swizzle).
// * Accumulation is chunked: the MMAs accumulate kChunk k-blocks (256 k) into TMEM, then the
//   converter warps add the chunk into fp32 registers (round-to-nearest) and the next chunk
//   restarts the TMEM accumulator. The tensor core's truncating fp32 accumulation therefore
//   only runs over F k-blocks whatever K is (the first design's error grew with K).
// * The factor is packed with NH = r~ rounded up to 8 (not 16): the main MMA covers
//   [U_hi | U_lo] with N = 2 NH, the cross MMA y_lo U_hi with N = NH (cta_group::1 MMAs take
//   N in steps of 8). r~ = 40: 120 MMA columns per k-step instead of 144.
// * Two accumulator buffers in TMEM alternate per chunk: the MMAs of chunk c + 1 run while the
//   converter warps add chunk c into their registers (the flush is deferred by one stage).
// Warp roles (10 warps; two CTAs per SM with 256 TMEM columns each, one with 512 for NH = 64):
//   warp 8      producer: TMA boxes of Y + bulk copy of the packed [U_hi | U_lo] k-block
//   warp 9      TMEM allocator + single-thread MMA issuer
//   warps 0-7   converters (y_lo into TMEM; warp w: TMEM lane quarter w & 3, k half w >> 2),
//               chunk flushes into register accumulators, and the epilogue stores
#include <algorithm>
#include <cstdlib>
#include <stdexcept>

#include "kernels.cuh"

namespace tkb {

namespace {

constexpr int kSConv = 8;                      // converter warps
constexpr int kSThreads = (kSConv + 2) * 32;   // + producer + MMA
constexpr int kSBK = 16;                       // k per pipeline stage (2 MMA k-steps of 8)

__host__ __device__ constexpr int round_up(int a, int b) { return (a + b - 1) / b * b; }

template <int NH, bool KM>
struct SCfg {
    static_assert(NH % 8 == 0 && NH >= 16 && NH <= 64, "NH: multiple of 8 in [16, 64]");
    static constexpr int TMEM = 512;                       // one CTA per SM, all of TMEM
    static constexpr int CN = NH;                          // N of the cross MMA (N steps of 8 are legal)
    static constexpr int DW = round_up(NH + CN, 16);       // accumulator columns per 128-row tile
    static constexpr int BM = 128;                         // rows per tile (one TMEM lane each)
    static constexpr int ND = 2;                           // accumulator buffers: chunk c -> buffer c & 1
    static constexpr int NA_FIT = (TMEM - ND * DW) / 32;   // [y_hi | y_lo] buffers, 32 columns each
    static constexpr int NA = NA_FIT > 8 ? 8 : NA_FIT;
    static_assert(NA >= 3, "TMEM budget");
    static constexpr int A_BASE = ND * DW;
    static constexpr int STAGE_B = 128 * NH;               // two k-steps of [U_hi | U_lo] (2 NH x 8 tf32 each)
    static constexpr int BST_FIT = (200 * 1024) / STAGE_B;
    static constexpr int BST = BST_FIT > 16 ? 16 : BST_FIT;  // factor ring depth
    static constexpr size_t BAR_BYTES = (2 * BST + 2 * NA + 4) * 8 + 16;
    static constexpr size_t smem = size_t(BST) * STAGE_B + BAR_BYTES;
    static constexpr int ACC = NH / 2;                     // accumulator columns per converter warp (its half)
    static constexpr int PF = 6;                           // stages of Y in flight per converter thread
};

// k-blocks (of 16) per accumulation chunk: the tensor core's truncating fp32 accumulation runs
// over at most kChunk * 16 k, then the chunk is added into fp32 registers (round to nearest)
constexpr int kChunk = 16;
// end of the chunk starting at k-block k0: kChunk blocks, the tail merged into the last full
// chunk when it would be shorter than `minlen` (every chunk has >= minlen blocks once nk >= minlen)
__device__ __forceinline__ int chunk_end(int k0, int nk, int minlen) {
    return nk - (k0 + kChunk) < minlen ? nk : k0 + kChunk;
}

__device__ __forceinline__ void sfence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void sfence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ void ld8(uint32_t taddr, float* v) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[e]);
}

__device__ __forceinline__ void ld4(uint32_t taddr, float* v) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = __uint_as_float(r[e]);
}

// UMMA shared-memory descriptors (sm_100): start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4
// [32,46), version 1 at bit 46, layout type [61,64): 0 none, 2 128B swizzle, 4 64B swizzle.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    return (uint64_t((saddr >> 4) & 0x3FFFu)) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
           (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (uint64_t(layout) << 61);
}

// Instruction descriptor: D f32, A/B tf32, B K-major, A MN-major if a_mn, M = 128, N = n.
__device__ __forceinline__ uint32_t sidesc(int n, bool a_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn ? (1u << 15) : 0u) | (uint32_t(n >> 3) << 17) |
           (uint32_t(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
                 : "memory");
}

// y_lo = y - trunc_tf32(y) (exact in fp32), rounded to nearest tf32 for the MMA
__device__ __forceinline__ uint32_t lo_bits(float y) {
    const float lo = y - __uint_as_float(__float_as_uint(y) & 0xFFFFE000u);
    return (__float_as_uint(lo) + 0x1000u) & 0xFFFFE000u;
}

// The converter thread of TMEM lane L and k half h loads its row's 8 k values of a stage
// straight from HBM (no shared-memory staging of Y: shared memory carries only the factor):
// KM = false: Y viewed as (P, K, Q); row p of tile (p0, q): y[p + k P + q P K] (a warp reads
//             32 consecutive p for one k: 128 coalesced bytes per load instruction);
//             out[p + r P + q P cols].
// KM = true:  Y viewed as Q rows of K contiguous values: 8 consecutive k = two 16-B loads;
//             out[row + r Q] (transposed output: the contracted mode moves last).
template <int NH, bool KM>
struct YLoader {
    const float* base = nullptr;  // this row's first element (null: a row beyond the tensor)
    int64_t kstride = 0;          // elements between consecutive k
    int64_t K = 0;
    __device__ __forceinline__ void load(int kc, int khalf, float (&v)[8]) const {
        const int64_t k0 = int64_t(kc) * kSBK + khalf * 8;
        if (!base) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = 0.f;
            return;
        }
        if constexpr (KM) {
            if (k0 + 8 <= K) {  // K % 4 == 0 and 16-B aligned rows
                const float4 a = __ldg(reinterpret_cast<const float4*>(base + k0));
                const float4 b = __ldg(reinterpret_cast<const float4*>(base + k0 + 4));
                v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = k0 + e < K ? __ldg(base + k0 + e) : 0.f;
            }
        } else {
            const float* p = base + k0 * kstride;
            if (k0 + 8 <= K) {  // warp-uniform: the K tail only in a tile's last stage
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = __ldg(p + e * kstride);
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = k0 + e < K ? __ldg(p + e * kstride) : 0.f;
            }
        }
    }
};

// First element of row L of tile t (null beyond the tensor), and of its output row: kept out of
// line (64-bit divisions, once per tile) so the unrolled stage loop stays within the register
// budget of 10-warp CTAs (168 per thread).
template <bool KM>
__device__ __noinline__ const float* tile_row(const float* y, int64_t t, int64_t tiles_p, int64_t P, int64_t K, int L) {
    if constexpr (KM) {
        const int64_t row = t * 128 + L;
        return row < P ? y + row * K : nullptr;
    } else {
        const int64_t q = t / tiles_p, p = (t - q * tiles_p) * 128 + L;
        return p < P ? y + q * P * K + p : nullptr;
    }
}
template <bool KM>
__device__ __noinline__ float* tile_out_row(float* out, int64_t t, int64_t tiles_p, int64_t P, int cols, int L) {
    int64_t q = 0, p0;
    if constexpr (KM) {
        p0 = t * 128;
    } else {
        q = t / tiles_p;
        p0 = (t - q * tiles_p) * 128;
    }
    return p0 + L < P ? out + q * P * cols + p0 + L : nullptr;
}

template <int NH, bool KM>
__global__ void __launch_bounds__(kSThreads, 1)
    ttm_stream_kernel(const float* __restrict__ y, const uint8_t* __restrict__ bpk, float* __restrict__ out,
                      int64_t P, int64_t K, int cols, int64_t tiles_p, int64_t ntiles) {
    using C = SCfg<NH, KM>;
    constexpr int BM = C::BM, NA = C::NA, BST = C::BST, PF = C::PF;
    extern __shared__ __align__(1024) uint8_t ssm[];
    uint8_t* sB = ssm;  // [BST][2 k-steps][2NH x 8] tf32 core matrices
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(BST) * C::STAGE_B);
    uint64_t* bfull = bars;              // [BST] producer -> MMA
    uint64_t* bempty = bfull + BST;      // [BST] MMA commit -> producer
    uint64_t* afull = bempty + BST;      // [NA]  converters (8) -> MMA
    uint64_t* aempty = afull + NA;       // [NA]  MMA commit -> converters
    uint64_t* dfull = aempty + NA;       // [2]   MMA commit (chunk done) -> converters
    uint64_t* dempty = dfull + 2;        // [2]   converters (8, chunk flushed) -> MMA
    uint32_t* tbase_sm = reinterpret_cast<uint32_t*>(dempty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = static_cast<int>((K + kSBK - 1) / kSBK);

    if (tid == 0) {
        for (int s = 0; s < BST; ++s) {
            mbar_init(&bfull[s], 1);
            mbar_init(&bempty[s], 1);
        }
        for (int a = 0; a < NA; ++a) {
            mbar_init(&afull[a], kSConv);
            mbar_init(&aempty[a], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&dfull[b], 1);
            mbar_init(&dempty[b], kSConv);
        }
        mbar_fence_init();
    }
    if (warp == kSConv + 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tbase_sm)),
                     "r"(C::TMEM));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    sfence_before();
    __syncthreads();
    sfence_after();
    const uint32_t tmem = *tbase_sm;

    if (warp == kSConv) {
        // ===== producer: the factor's k-blocks (the only shared-memory operand) =====
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int kc = 0; kc < nk; ++kc) {
                    mbar_wait(&bempty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&bfull[s], C::STAGE_B);
                    bulk_g2s(sB + size_t(s) * C::STAGE_B, bpk + size_t(kc) * C::STAGE_B, C::STAGE_B, &bfull[s]);
                    if (++s == BST) s = 0, ph ^= 1;
                }
            }
        }
    } else if (warp == kSConv + 1) {
        // ===== MMA issuer: D[0:2NH] += y_hi [U_hi | U_lo], D[NH:2NH] += y_lo U_hi =====
        if (lane == 0) {
            const uint32_t id_main = sidesc(2 * NH, false), id_cross = sidesc(C::CN, false);
            int s = 0, a = 0;
            uint32_t ph = 0, aph = 0, ch = 0;
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int k0 = 0, k1 = 0; k0 < nk; k0 = k1, ++ch) {
                    k1 = chunk_end(k0, nk, PF);
                    const int b = ch & 1;
                    if (ch >= 2) {  // this buffer's previous chunk has been added into the registers
                        mbar_wait(&dempty[b], ((ch >> 1) - 1) & 1);
                        sfence_after();
                    }
                    const uint32_t dm = tmem + uint32_t(b * C::DW);
                    for (int kc = k0; kc < k1; ++kc) {
                        mbar_wait(&bfull[s], ph);
                        mbar_wait(&afull[a], aph);
                        sfence_after();
                        const uint32_t bs = smem_u32(sB + size_t(s) * C::STAGE_B);
                        const uint32_t ahi = tmem + uint32_t(C::A_BASE + a * 32);
#pragma unroll
                        for (int ks = 0; ks < 2; ++ks) {
                            const uint64_t bd = sdesc(bs + ks * (64 * NH), 128, 256, 0);
                            mma_ts(dm, ahi + ks * 8, bd, id_main, (kc > k0 || ks > 0) ? 1u : 0u);
                            mma_ts(dm + NH, ahi + 16 + ks * 8, bd, id_cross, 1u);
                        }
                        commit(&aempty[a]);
                        commit(&bempty[s]);
                        if (++s == BST) s = 0, ph ^= 1;
                        if (++a == NA) a = 0, aph ^= 1;
                    }
                    commit(&dfull[b]);
                }
            }
        }
    } else {
        // ===== converters (warps 0-7): lane quarter warp & 3, k half warp >> 2 =====
        const int quarter = warp & 3, khalf = warp >> 2;
        const int L = quarter * 32 + lane;  // TMEM lane = row of the 128-row tile
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        constexpr int ACC = C::ACC;
        const int c0 = khalf * (NH / 2);
        float acc[ACC];
#pragma unroll
        for (int e = 0; e < ACC; ++e) acc[e] = 0.f;
        // (tile, k-block) sequence of this CTA, walked PF stages ahead by the loads
        auto row_of = [&](int64_t t) {
            YLoader<NH, KM> ld;
            ld.K = K;
            ld.base = tile_row<KM>(y, t, tiles_p, P, K, L);
            ld.kstride = KM ? 1 : P;
            return ld;
        };
        float pf[PF][8];
        // prefetch cursor: (tile, k-block) PF stages ahead of the consumer, same order
        int64_t tl = blockIdx.x;
        int kl = 0;
        YLoader<NH, KM> ldl = row_of(tl);
        auto advance_load = [&](float (&v)[8]) {
            if (tl < ntiles) {
                ldl.load(kl, khalf, v);
                if (++kl == nk) {
                    kl = 0;
                    tl += gridDim.x;
                    if (tl < ntiles) ldl = row_of(tl);
                }
            }
        };
#pragma unroll
        for (int i = 0; i < PF; ++i) advance_load(pf[i]);
        int a = 0;
        uint32_t aph = 0, ch = 0;
        auto flush = [&](uint32_t c) {
            const int b = c & 1;
            mbar_wait(&dfull[b], (c >> 1) & 1);
            sfence_after();
            const uint32_t base = tmem + lane_off + uint32_t(b * C::DW + c0);
#pragma unroll
            for (int cc = 0; cc < ACC; cc += 4) {  // 4 main + 4 cross columns at a time (few temporaries)
                float m[4], x[4];
                ld4(base + cc, m);
                ld4(base + NH + cc, x);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[cc + e] += m[e] + x[e];
            }
            sfence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&dempty[b]);
        };
        auto store = [&](float* orow) {
            if (orow) {
#pragma unroll
                for (int e = 0; e < ACC; ++e)
                    if (c0 + e < cols) orow[int64_t(c0 + e) * P] = acc[e];
            }
#pragma unroll
            for (int e = 0; e < ACC; ++e) acc[e] = 0.f;
        };
        // consumer: this CTA's stages in order, unrolled by PF so the prefetch ring is indexed
        // statically (stage g lives in pf[g % PF]). Every chunk has >= PF stages, so at most one
        // ends per group of PF; it is added into the registers at the end of the NEXT group
        // (its MMAs are long done by then; the MMA needs the buffer again a whole chunk later).
        int64_t t = blockIdx.x;
        int kc = 0, kend = chunk_end(0, nk, PF);
        const int64_t total = t < ntiles ? ((ntiles - 1 - t) / gridDim.x + 1) * int64_t(nk) : 0;
        bool pending = false;
        uint32_t pend = 0;
        float* pend_row = nullptr;
        bool pend_tile = false;
        for (int64_t g0 = 0; g0 < total; g0 += PF) {
            bool ended = false, ended_tile = false;
            uint32_t ended_ch = 0;
            float* ended_row = nullptr;
#pragma unroll
            for (int i = 0; i < PF; ++i) {
                if (g0 + i < total) {
                    uint32_t hi[8], lo[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const float v = pf[i][e];
                        const uint32_t hb = (__float_as_uint(v) + 0x1000u) & 0xFFFFE000u;  // round to nearest tf32
                        hi[e] = hb;
                        lo[e] = __float_as_uint(v - __uint_as_float(hb));                 // exact residual
                    }
                    advance_load(pf[i]);  // refill the slot PF stages ahead
                    mbar_wait(&aempty[a], aph ^ 1);
                    sfence_after();
                    st8(tmem + lane_off + uint32_t(C::A_BASE + a * 32 + khalf * 8), hi);
                    st8(tmem + lane_off + uint32_t(C::A_BASE + a * 32 + 16 + khalf * 8), lo);
                    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                    sfence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&afull[a]);
                    if (++a == NA) a = 0, aph ^= 1;
                    if (kc + 1 == kend) {  // chunk end
                        ended = true;
                        ended_ch = ch++;
                        if (kend == nk) {  // tile end: the rows are stored once this chunk is added
                            ended_tile = true;
                            ended_row = tile_out_row<KM>(out, t, tiles_p, P, cols, L);
                        }
                    }
                    if (++kc == nk) {
                        kc = 0;
                        t += gridDim.x;
                        kend = chunk_end(0, nk, PF);
                    } else if (kc == kend) {
                        kend = chunk_end(kc, nk, PF);
                    }
                }
            }
            if (pending) {
                flush(pend);
                if (pend_tile) store(pend_row);
                pending = false;
            }
            if (ended) {
                pending = true;
                pend = ended_ch;
                pend_tile = ended_tile;
                pend_row = ended_row;
            }
        }
        if (pending) {  // this CTA's last chunk
            flush(pend);
            if (pend_tile) store(pend_row);
        }
    }
    sfence_before();
    __syncthreads();
    if (warp == kSConv + 1) {
        sfence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(C::TMEM));
    }
}

// [U_hi | U_lo] of a column-major fp64 factor (rows x cols, ld), tf32 in the UMMA K-major
// no-swizzle core-matrix layout: per k-step of 8 rows of U, 2NH n-rows of 8 k (16-B core
// matrix rows, 8-row groups 256 B apart, the two 4-k halves 128 B apart).
__global__ void pack_stream_kernel(const double* __restrict__ u, int64_t ld, int64_t rows, int cols, int nh,
                                   int64_t ksteps, uint32_t* __restrict__ out) {
    const int64_t n_el = ksteps * 2 * nh * 8;
    for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n_el; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t g = t / (2 * nh * 8);
        const int rem = static_cast<int>(t % (2 * nh * 8));
        const int n = rem / 8, kk = rem % 8;
        const int64_t k = g * 8 + kk;
        const int r = n < nh ? n : n - nh;
        const float uf = (k < rows && r < cols) ? static_cast<float>(u[k + int64_t(r) * ld]) : 0.f;
        uint32_t h;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(uf));
        uint32_t v = h;
        if (n >= nh) asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(v) : "f"(uf - __uint_as_float(h)));
        const int64_t byte = g * (64 * nh) + (n / 8) * 256 + (kk / 4) * 128 + (n % 8) * 16 + (kk % 4) * 4;
        out[byte / 4] = v;
    }
}

template <int NH, bool KM>
void launch_stream(const float* in, const uint8_t* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                   cudaStream_t s) {
    using C = SCfg<NH, KM>;
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(ttm_stream_kernel<NH, KM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(C::smem)));
        attr = true;
    }
    int64_t tiles_p, ntiles, rows;
    if constexpr (KM) {  // Q rows of K contiguous values
        tiles_p = (Q + C::BM - 1) / C::BM;
        ntiles = tiles_p;
        rows = Q;
    } else {
        tiles_p = (P + C::BM - 1) / C::BM;
        ntiles = tiles_p * Q;
        rows = P;
    }
    const int64_t grid = std::min<int64_t>(ntiles, 148);
    TK_MAXSMEM((ttm_stream_kernel<NH, KM>));
    ttm_stream_kernel<NH, KM><<<static_cast<unsigned>(grid), kSThreads, C::smem, s>>>(in, bpk, out, rows, K, cols,
                                                                                     tiles_p, ntiles);
    TK_LAUNCH_CHECK();
}

inline int stream_nh(int cols) { return std::max(16, (cols + 7) / 8 * 8); }

}  // namespace

bool stream_ttm_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("TENKIT_STREAM");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool stream_ttm_supported(const float* in, float* out, int64_t P, int64_t K, int64_t Q, int cols) {
    if (reinterpret_cast<uintptr_t>(in) % 16 != 0 || reinterpret_cast<uintptr_t>(out) % 16 != 0) return false;
    if (cols < 1 || cols > kMaxRank || K < 8 * kSBK) return false;  // >= PF k-blocks per tile
    if (P == 1) return K % 4 == 0 && (Q + 127) / 128 >= 2 * 148;    // K-major: >= two waves of 128-row tiles
    return P % 4 == 0 && P >= 128 && (P + 127) / 128 * Q >= 2 * 148;
}

int64_t stream_pack_bytes(int64_t rows, int cols) {
    const int64_t ksteps = (rows + kSBK - 1) / kSBK * 2;
    return ksteps * 64 * stream_nh(cols);
}

void launch_pack_stream(const double* u, int64_t ld, int64_t rows, int cols, void* out, cudaStream_t s) {
    require(cols >= 1 && cols <= kMaxRank, "ttm: factor column count must be in [1, 64]");
    const int64_t ksteps = (rows + kSBK - 1) / kSBK * 2;
    const int nh = stream_nh(cols);
    const int64_t n = ksteps * 2 * nh * 8;
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)));
    TK_MAXSMEM(pack_stream_kernel);
    pack_stream_kernel<<<grid, 256, 0, s>>>(u, ld, rows, cols, nh, ksteps, static_cast<uint32_t*>(out));
    TK_LAUNCH_CHECK();
}

// P == 1: contraction over mode 0, transposed output out[q + r Q]; else out[p + r P + q P cols].
void launch_ttm_stream(const float* in, const void* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                       cudaStream_t s) {
    const uint8_t* b = static_cast<const uint8_t*>(bpk);
    const int nh = stream_nh(cols);
#define TK_STREAM_CASE(N)                                                   \
    case N:                                                                 \
        if (P == 1) launch_stream<N, true>(in, b, out, P, K, Q, cols, s);   \
        else launch_stream<N, false>(in, b, out, P, K, Q, cols, s);         \
        break;
    switch (nh) {
        TK_STREAM_CASE(16)
        TK_STREAM_CASE(24)
        TK_STREAM_CASE(32)
        TK_STREAM_CASE(40)
        TK_STREAM_CASE(48)
        TK_STREAM_CASE(56)
        TK_STREAM_CASE(64)
        default: throw InvalidArgument("tenkit: ttm: factor column count must be in [1, 64]");
    }
#undef TK_STREAM_CASE
}

}  // namespace tkb
