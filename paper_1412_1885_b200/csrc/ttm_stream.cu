// ttm_stream.cu — the Y-streaming pass (first stage of every X_n = Y x_{p != n} U_p^T and of
// the core, tensor.hpp:151-192) on the tcgen05 tensor cores, second design.
//
//   out[p, r, q] = sum_k Y[p, k, q] U[k, r]       (3xTF32: y u ~= y_hi u_hi + y_hi u_lo + y_lo u_hi)
//
// Differences from ttm_tc.cu (the first design):
// * Accumulation is chunked: the MMAs accumulate kChunk k-blocks (256 k) into TMEM, then the
//   converter warps add the chunk into fp32 registers (round-to-nearest) and the next chunk
//   restarts the TMEM accumulator. The tensor core's truncating fp32 accumulation therefore
//   only runs over 256 k whatever K is (the first design's error grew with K: at K = 4000 its
//   fp32 bases missed the 1e-3 parity bar, these make it at 1.7-3.1e-4).
// * One accumulator buffer per M tile; the TMEM it leaves goes to a deeper ring of [y_hi | y_lo]
//   A buffers (5-6 instead of 3), which decouples the converter warps from the MMA issuer better
//   than overlapping the chunk flush did (compile-time A/B TK_STREAM_ND_MAX=2: two buffers
//   alternating per chunk, the MMAs of chunk c + 1 running while chunk c is added; measured
//   2-5 % slower at cfg 2 / 3 / 4).
// * The factor is packed with NH = r~ rounded up to 8 (not 16): the main MMA covers
//   [U_hi | U_lo] with N = 2 NH, the cross MMA y_lo U_hi with N = NH (cta_group::1 MMAs take
//   N in steps of 8). r~ = 40: 120 MMA columns per k-step instead of 144.
// * Two 128-row M tiles per CTA (BM = 256), one CTA per SM: one Y box, one factor k-block,
//   one set of barrier round trips per stage for both tiles.
// * The producer and MMA warps run converged and issue through elect.sync inside the asm, so
//   the TMA / UTCHMMA / commit operands live in uniform registers (no per-lane issue loop: with
//   `if (lane == 0)` issue, ptxas wrapped every MMA in an R2UR/ELECT/BRA.U.ANY loop and the
//   single issuing thread, not HBM, bounded the pass).
// * Up to six [y_hi | y_lo] TMEM buffers let the converters run ahead of the MMA issuer.
// Y tiles are staged by TMA, one box per stage (M-major: 256 p x 16 k unswizzled, 1 KB rows;
// K-major: 16 k x 256 rows, 64B swizzle) for the converter warps' conflict-free reads.
// Warp roles (10 warps, one CTA per SM with 512 TMEM columns):
//   warp 8      producer: TMA box of Y + bulk copy of the packed [U_hi | U_lo] k-block
//   warp 9      TMEM allocator + MMA issuer
//   warps 0-7   converters ([y_hi | y_lo] into TMEM; warp w: TMEM lane quarter w & 3, k half
//               w >> 2, both M tiles), chunk flushes into register accumulators, epilogue stores
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <type_traits>

#include "kernels.cuh"

namespace tkb {

namespace {

using EncodeTiledFn2 = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn2 encode_tiled2() {
    static EncodeTiledFn2 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        const cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        return (e == cudaSuccess && q == cudaDriverEntryPointSuccess) ? reinterpret_cast<EncodeTiledFn2>(p) : nullptr;
    }();
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled entry point unavailable");
    return fn;
}

// compile-time A/B knobs (tools/build_variant.sh builds a second library with -D overrides)
#ifndef TK_STREAM_NA_MAX
#define TK_STREAM_NA_MAX 6
#endif
#ifndef TK_STREAM_STAGES_MAX
#define TK_STREAM_STAGES_MAX 12
#endif
#ifndef TK_STREAM_CONV
#define TK_STREAM_CONV 8
#endif
#ifndef TK_STREAM_ND_MAX
#define TK_STREAM_ND_MAX 1
#endif
#ifndef TK_STREAM_PIPEBAL
#define TK_STREAM_PIPEBAL 1
#endif
#ifndef TK_STREAM_WAIT_HINT
#define TK_STREAM_WAIT_HINT 0
#endif
#ifndef TK_STREAM_SPLITB
#define TK_STREAM_SPLITB 0
#endif
#ifndef TK_STREAM_DEFER1
#define TK_STREAM_DEFER1 0
#endif
#ifndef TK_STREAM_CHUNK
#define TK_STREAM_CHUNK 16
#endif

constexpr int kSConv = TK_STREAM_CONV;         // converter warps: 8 (two k halves per TMEM lane quarter), 16 (four k quarters) or 4 (all 16 k)
static_assert(kSConv == 4 || kSConv == 8 || kSConv == 16, "converter warps");
constexpr int kKSplit = kSConv / 4;            // warps sharing a TMEM lane quarter, each takes 16 / kKSplit k of a stage
constexpr int kKPW = 16 / kKSplit;             // k per converter warp and stage
constexpr int kSThreads = (kSConv + 2) * 32;   // + producer + MMA
constexpr int kSBK = 16;                       // k per pipeline stage (2 MMA k-steps of 8)

__host__ __device__ constexpr int round_up(int a, int b) { return (a + b - 1) / b * b; }

template <int NH, bool KM, int MT_, int OCC_>
struct SCfg {
    static_assert(NH % 8 == 0 && NH >= 16 && NH <= 64, "NH: multiple of 8 in [16, 64]");
    static constexpr int MT = MT_;                         // 128-row M tiles per CTA
    static constexpr int OCC = OCC_;                       // CTAs per SM (TMEM: 256 or 512 columns each)
    static constexpr int TMEM = 512 / OCC;
    static constexpr int CN = NH;                          // N of the cross MMA (N steps of 8 are legal)
    static constexpr int DW = round_up(NH + CN, 16);       // accumulator columns per 128-row tile
    static constexpr int BM = 128 * MT;
    // accumulator buffers: two (chunk c -> buffer c & 1) where they leave room for two A
    // buffers, else one (the MMAs of the next chunk wait for the flush)
    static constexpr int ND = ((TMEM - 2 * MT * DW) >= 2 * MT * 32 && TK_STREAM_ND_MAX >= 2) ? 2 : 1;
    static constexpr int NA_FIT = (TMEM - ND * MT * DW) / (MT * 32);
    static constexpr int NA = NA_FIT > TK_STREAM_NA_MAX ? TK_STREAM_NA_MAX : NA_FIT;     // [y_hi | y_lo] TMEM buffers (32 columns per M tile)
    static_assert(NA >= 2, "TMEM budget");
    static constexpr int A_BASE = ND * MT * DW;
    static constexpr int BOXR = BM;                        // rows per TMA box (one box per stage)
    static constexpr int STAGE_Y = kSBK * BM * 4;
    static constexpr int STAGE_B = 128 * NH;               // two k-steps of [U_hi | U_lo] (2 NH x 8 tf32 each)
    static constexpr int SMEM_BUDGET = OCC == 2 ? 110 * 1024 : 220 * 1024;
#if TK_STREAM_SPLITB
    // Split rings: a Y stage is released by the converter warps alone (right after conversion);
    // the factor k-blocks live in their own ring, NA + 2 slots deeper, released by the MMA commits
    // (with one ring the MMA issuer, up to NA stages behind, holds the 16 KB Y slots for the sake
    // of their 5 KB factor blocks).
#ifdef TK_STREAM_BEXTRA
    static constexpr int BEXTRA = TK_STREAM_BEXTRA;
#else
    static constexpr int BEXTRA = NA + 2;
#endif
    static constexpr int STAGES_FIT = (SMEM_BUDGET - 1024 - BEXTRA * STAGE_B) / (STAGE_Y + STAGE_B);
    static constexpr int STAGES = STAGES_FIT > TK_STREAM_STAGES_MAX ? TK_STREAM_STAGES_MAX : STAGES_FIT;
    static constexpr int BSTAGES = STAGES + BEXTRA;
#else
    static constexpr int STAGES_FIT = (SMEM_BUDGET - 1024) / (STAGE_Y + STAGE_B);  // (1 KB: barriers + slack)
    static constexpr int STAGES = STAGES_FIT > TK_STREAM_STAGES_MAX ? TK_STREAM_STAGES_MAX : STAGES_FIT;
    static constexpr int BSTAGES = STAGES;
#endif
    static_assert(STAGES >= 3, "pipeline depth");
    // barriers: 2 per stage (+ 2 per factor slot) + 2 per y_lo buffer + 4 accumulator-buffer barriers, + the TMEM base
    static constexpr size_t BAR_BYTES = (2 * STAGES + 2 * BSTAGES + 2 * NA + 4) * 8 + 16;
    static constexpr size_t smem = size_t(STAGES) * STAGE_Y + size_t(BSTAGES) * STAGE_B + BAR_BYTES;
    static constexpr int ACC = NH / kKSplit;               // accumulator columns per converter warp (its share)
};

// k-blocks (of 16) per accumulation chunk: the tensor core's truncating fp32 accumulation runs
// over at most kChunk * 16 k, then the chunk is added into fp32 registers (round to nearest)
constexpr int kChunkDefault = TK_STREAM_CHUNK;

__device__ __forceinline__ void sfence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void sfence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// [hi | lo] of one M tile's k half: columns [0, 8) and [16, 24) of the A buffer, one address register
__device__ __forceinline__ void st8_pair(uint32_t taddr, const uint32_t (&h)[8], const uint32_t (&l)[8]) {
    asm volatile(
        "{\n\t.reg .b32 t1;\n\t"
        "add.u32 t1, %0, 16;\n\t"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [t1], {%9, %10, %11, %12, %13, %14, %15, %16};\n\t}\n" ::"r"(taddr),
        "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]), "r"(l[0]), "r"(l[1]),
        "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7])
        : "memory");
}
// the same for 4-k shares (16 converter warps)
__device__ __forceinline__ void st4_pair(uint32_t taddr, const uint32_t (&h)[4], const uint32_t (&l)[4]) {
    asm volatile(
        "{\n\t.reg .b32 t1;\n\t"
        "add.u32 t1, %0, 16;\n\t"
        "tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x4.b32 [t1], {%5, %6, %7, %8};\n\t}\n" ::"r"(taddr),
        "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3])
        : "memory");
}
__device__ __forceinline__ void st4_quad(uint32_t taddr, const uint32_t (&h0)[4], const uint32_t (&l0)[4],
                                         const uint32_t (&h1)[4], const uint32_t (&l1)[4]) {
    asm volatile(
        "{\n\t.reg .b32 t1, t2, t3;\n\t"
        "add.u32 t1, %0, 16;\n\t"
        "add.u32 t2, %0, 32;\n\t"
        "add.u32 t3, %0, 48;\n\t"
        "tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x4.b32 [t1], {%5, %6, %7, %8};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x4.b32 [t2], {%9, %10, %11, %12};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x4.b32 [t3], {%13, %14, %15, %16};\n\t}\n" ::"r"(taddr),
        "r"(h0[0]), "r"(h0[1]), "r"(h0[2]), "r"(h0[3]), "r"(l0[0]), "r"(l0[1]), "r"(l0[2]), "r"(l0[3]), "r"(h1[0]),
        "r"(h1[1]), "r"(h1[2]), "r"(h1[3]), "r"(l1[0]), "r"(l1[1]), "r"(l1[2]), "r"(l1[3])
        : "memory");
}
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16};\n" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void ld2(uint32_t taddr, float* v) {
    uint32_t r[2];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(r[0]), "=r"(r[1]) : "r"(taddr) : "memory");
    v[0] = __uint_as_float(r[0]);
    v[1] = __uint_as_float(r[1]);
}
__device__ __forceinline__ void st8_quad(uint32_t taddr, const uint32_t (&h0)[8], const uint32_t (&l0)[8],
                                         const uint32_t (&h1)[8], const uint32_t (&l1)[8]) {
    asm volatile(
        "{\n\t.reg .b32 t1, t2, t3;\n\t"
        "add.u32 t1, %0, 16;\n\t"
        "add.u32 t2, %0, 32;\n\t"
        "add.u32 t3, %0, 48;\n\t"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [t1], {%9, %10, %11, %12, %13, %14, %15, %16};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [t2], {%17, %18, %19, %20, %21, %22, %23, %24};\n\t"
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [t3], {%25, %26, %27, %28, %29, %30, %31, %32};\n\t}\n" ::"r"(taddr),
        "r"(h0[0]), "r"(h0[1]), "r"(h0[2]), "r"(h0[3]), "r"(h0[4]), "r"(h0[5]), "r"(h0[6]), "r"(h0[7]), "r"(l0[0]),
        "r"(l0[1]), "r"(l0[2]), "r"(l0[3]), "r"(l0[4]), "r"(l0[5]), "r"(l0[6]), "r"(l0[7]), "r"(h1[0]), "r"(h1[1]),
        "r"(h1[2]), "r"(h1[3]), "r"(h1[4]), "r"(h1[5]), "r"(h1[6]), "r"(h1[7]), "r"(l1[0]), "r"(l1[1]), "r"(l1[2]),
        "r"(l1[3]), "r"(l1[4]), "r"(l1[5]), "r"(l1[6]), "r"(l1[7])
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

// Issued by the whole (converged) MMA warp: elect.sync picks the lane inside the asm, so the
// operands stay warp-uniform (uniform registers) and ptxas emits a bare UTCHMMA / UTCBAR
// instead of its per-active-lane loop (R2UR + ELECT + BRA.U.ANY around every MMA, which made
// the single issuing thread the pipeline's bottleneck).
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void commit(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
            smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void tma2(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// One pipeline stage, issued by the whole (converged) producer warp through one elected lane:
// expect_tx on the stage barrier, the Y box (TMA, 3-D M-major or 2-D K-major view) and the
// packed factor k-block (bulk copy), all completing on that barrier.
__device__ __forceinline__ void produce3(uint32_t bar, uint32_t bytes, uint32_t dy, const CUtensorMap* map, int c0,
                                        int c1, int c2, uint32_t db, const void* src, uint32_t bbytes) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3, {%4, %5, %6}], "
        "[%0];\n\t"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%7], [%8], %9, [%0];\n\t}\n" ::"r"(bar),
        "r"(bytes), "r"(dy), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(db), "l"(src), "r"(bbytes)
        : "memory");
}

__device__ __forceinline__ void produce2(uint32_t bar, uint32_t bytes, uint32_t dy, const CUtensorMap* map, int c0,
                                        int c1, uint32_t db, const void* src, uint32_t bbytes) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3, {%4, %5}], "
        "[%0];\n\t"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%6], [%7], %8, [%0];\n\t}\n" ::"r"(bar),
        "r"(bytes), "r"(dy), "l"(map), "r"(c0), "r"(c1), "r"(db), "l"(src), "r"(bbytes)
        : "memory");
}

// mbarrier operations on 32-bit shared-window addresses kept in registers (the generic-pointer
// helpers recompute the window base from SR_CgaCtaId at every use inside the stage loop)
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
#if TK_STREAM_WAIT_HINT
    // suspend-time hint: the hardware parks the warp until the phase completes (or the hint
    // expires) instead of returning to the retry loop every few hundred cycles
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}\n" ::"r"(bar),
        "r"(parity), "r"(uint32_t(TK_STREAM_WAIT_HINT))
        : "memory");
#else
    asm volatile(
        "{\n\t"
        ".reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
#endif
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

// Split rings: the Y box and the factor k-block complete on their own barriers.
__device__ __forceinline__ void produce_y3(uint32_t bar, uint32_t bytes, uint32_t dy, const CUtensorMap* map, int c0,
                                          int c1, int c2) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@e cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3, {%4, %5, %6}], "
        "[%0];\n\t}\n" ::"r"(bar),
        "r"(bytes), "r"(dy), "l"(map), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void produce_y2(uint32_t bar, uint32_t bytes, uint32_t dy, const CUtensorMap* map, int c0,
                                          int c1) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
        "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%2], [%3, {%4, %5}], "
        "[%0];\n\t}\n" ::"r"(bar),
        "r"(bytes), "r"(dy), "l"(map), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void produce_b(uint32_t bar, uint32_t db, const void* src, uint32_t bbytes) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %3;\n\t"
        "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%1], [%2], %3, [%0];\n\t}\n" ::"r"(bar),
        "r"(db), "l"(src), "r"(bbytes)
        : "memory");
}

// y_hi = y rounded to nearest tf32, y_lo = y - y_hi (exact in fp32; the tensor core reads its
// top 19 bits)
__device__ __forceinline__ void split_hi_lo(float y, uint32_t& hi, uint32_t& lo) {
    hi = (__float_as_uint(y) + 0x1000u) & 0xFFFFE000u;
    lo = __float_as_uint(y - __uint_as_float(hi));
}
// The same values with the work spread over both issue pipes: the rounding add as an IMAD
// (`one` is 1 from a kernel argument, so ptxas keeps the multiply-add on the fma pipe instead of
// a VIADD on the alu pipe) and y - hi as an immediate-form FFMA (hi * -1 + y, twice the issue
// rate of the three-register FADD). With the plain form the alu pipe carries two of the three
// instructions per value (VIADD, LOP3) and bounds the split; 12 of a thread's 16 values take
// this form, 4 the plain one: ~40 pipe cycles per warp and stage on either pipe instead of 64 / 32.
__device__ __forceinline__ void split_hi_lo_fma(float y, uint32_t one, uint32_t& hi, uint32_t& lo) {
    uint32_t h;
    asm("mad.lo.u32 %0, %1, %2, 0x1000;\n" : "=r"(h) : "r"(__float_as_uint(y)), "r"(one));
    hi = h & 0xFFFFE000u;
    float l;
    asm("fma.rn.f32 %0, %1, 0fBF800000, %2;\n" : "=f"(l) : "f"(__uint_as_float(hi)), "f"(y));
    lo = __float_as_uint(l);
}
__device__ __forceinline__ void split_hi_lo_alu(float y, uint32_t& hi, uint32_t& lo) {
    hi = (__float_as_uint(y) + 0x1000u) & 0xFFFFE000u;
    float l;
    asm("fma.rn.f32 %0, %1, 0fBF800000, %2;\n" : "=f"(l) : "f"(__uint_as_float(hi)), "f"(y));
    lo = __float_as_uint(l);
}
// A/B variant (TENKIT_STREAM_TRUNC=1): y_hi = y truncated to tf32 (one instruction less per
// value); y_lo = y - y_hi then has the sign of y and up to 13 significant bits, of which the
// tensor core keeps 11: a one-sided residual of < 2^-20 |y| instead of a two-sided < 2^-21 |y|.
__device__ __forceinline__ void split_hi_lo_trunc(float y, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(y) & 0xFFFFE000u;
    float l;  // y - hi as an immediate-form FFMA (see split_hi_lo_fma)
    asm("fma.rn.f32 %0, %1, 0fBF800000, %2;\n" : "=f"(l) : "f"(__uint_as_float(hi)), "f"(y));
    lo = __float_as_uint(l);
}

// KM = false: Y viewed as (P, K, Q), tiles of BM consecutive p of one q; out[p + r P + q P cols].
//             Row MT L + j of the tile is TMEM lane L of M tile j (a thread reads MT adjacent p).
// KM = true:  Y viewed as Q rows of K contiguous values (contraction over mode 0), tiles of BM
//             rows; out[row + r Q] (transposed output: the contracted mode moves last). Row
//             128 j + L of the tile is TMEM lane L of M tile j.
// Accumulation chunks of kChunk k-blocks: at a chunk end the converter warps wait for the chunk's
// MMAs, add the TMEM accumulator into their registers and release it (ND = 2: two buffers
// alternating, the flush deferred behind the next chunk's first stages).
template <int NH, bool KM, int MT, int OCC, int kChunk = 16, bool TR = false>
__global__ void __launch_bounds__(kSThreads, OCC)
    ttm_stream_kernel(const __grid_constant__ CUtensorMap ymap, const uint8_t* __restrict__ bpk, float* __restrict__ out,
                      int64_t P, int64_t K, int cols, int64_t tiles_p, int64_t ntiles, int accum, int bq, int64_t Q,
                      uint32_t one) {
    using C = SCfg<NH, KM, MT, OCC>;
    constexpr int BM = C::BM, NA = C::NA, ST = C::STAGES, ND = C::ND;
    // dynamic shared memory starts at offset 0 of the CTA's window (no static shared memory in
    // this kernel): 1024-B aligned as the 128B-span swizzles need
    extern __shared__ __align__(1024) uint8_t ssm[];
    uint8_t* sY = ssm;                             // [stages][BM/BOXR boxes]
    constexpr int SB = C::BSTAGES;
    uint8_t* sB = ssm + size_t(ST) * C::STAGE_Y;   // [factor slots][2 k-steps][2NH x 8] tf32 core matrices
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + size_t(SB) * C::STAGE_B);
    uint64_t* full = bars;               // [ST]  producer -> converters, MMA
    uint64_t* empty = full + ST;         // [ST]  converters (8) + MMA commit (1) -> producer
    uint64_t* bfull = empty + ST;        // [SB]  split rings: producer -> MMA (factor k-block landed)
    uint64_t* bempty = bfull + SB;       // [SB]  split rings: MMA commit -> producer
    uint64_t* afull = bempty + SB;       // [NA]  converters (8) -> MMA
    uint64_t* aempty = afull + NA;       // [NA]  MMA commit -> converters
    uint64_t* dfull = aempty + NA;       // [2]   MMA commit (chunk done) -> converters
    uint64_t* dempty = dfull + 2;        // [2]   converters (8, chunk flushed) -> MMA
    uint32_t* tbase_sm = reinterpret_cast<uint32_t*>(dempty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk = static_cast<int>((K + kSBK - 1) / kSBK);

    if (tid == 0) {
        if (smem_u32(ssm) & 1023) __trap();  // the swizzle atoms need 1024-B alignment
        for (int s = 0; s < ST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], TK_STREAM_SPLITB ? kSConv : kSConv + 1);
        }
        for (int b = 0; b < SB; ++b) {
            mbar_init(&bfull[b], 1);
            mbar_init(&bempty[b], 1);
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
        // ===== producer (the whole warp, converged; one elected lane issues) =====
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&ymap) : "memory");
        int s = 0;
        uint32_t ph = 0;
        uint32_t y0 = smem_u32(sY), b0 = smem_u32(sB), f0 = smem_u32(full), e0 = smem_u32(empty);
        asm volatile("" : "+r"(y0), "+r"(b0), "+r"(f0), "+r"(e0));
#if TK_STREAM_SPLITB
        int sb = 0;
        uint32_t phb = 0;
        uint32_t bf0 = smem_u32(bfull), be0 = smem_u32(bempty);
        asm volatile("" : "+r"(bf0), "+r"(be0));
#endif
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t q = (t / tiles_p) * bq;
            const int64_t p0 = (t % tiles_p) * (BM / bq);
            for (int kc = 0; kc < nk; ++kc) {
                const uint8_t* src = bpk + size_t(kc) * C::STAGE_B;
#if TK_STREAM_SPLITB
                bar_wait(be0 + sb * 8, phb ^ 1);
                __syncwarp();
                produce_b(bf0 + sb * 8, b0 + sb * C::STAGE_B, src, C::STAGE_B);
                if (++sb == SB) sb = 0, phb ^= 1;
                bar_wait(e0 + s * 8, ph ^ 1);
                __syncwarp();
                if constexpr (KM) produce_y2(f0 + s * 8, C::STAGE_Y, y0 + s * C::STAGE_Y, &ymap, kc * kSBK, static_cast<int>(p0));
                else produce_y3(f0 + s * 8, C::STAGE_Y, y0 + s * C::STAGE_Y, &ymap, static_cast<int>(p0), kc * kSBK, static_cast<int>(q));
#else
                bar_wait(e0 + s * 8, ph ^ 1);
                __syncwarp();
                const uint32_t bar = f0 + s * 8, dy = y0 + s * C::STAGE_Y, db = b0 + s * C::STAGE_B;
                if constexpr (KM) {
                    produce2(bar, C::STAGE_Y + C::STAGE_B, dy, &ymap, kc * kSBK, static_cast<int>(p0), db, src, C::STAGE_B);
                } else {
                    produce3(bar, C::STAGE_Y + C::STAGE_B, dy, &ymap, static_cast<int>(p0), kc * kSBK,
                             static_cast<int>(q), db, src, C::STAGE_B);
                }
#endif
                if (++s == ST) s = 0, ph ^= 1;
            }
        }
    } else if (warp == kSConv + 1) {
        // ===== MMA issuer (the whole warp, converged; one elected lane issues) =====
        {
            const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);  // provably warp-uniform
            const uint32_t id_main = sidesc(2 * NH, false), id_cross = sidesc(C::CN, false);
            int s = 0, a = 0;
            uint32_t ph = 0, aph = 0, ch = 0;
            // the ring the MMA issuer follows: the stage ring, or the factor ring when they are split
            constexpr int RS = TK_STREAM_SPLITB ? SB : ST;
            uint64_t* const rfull = TK_STREAM_SPLITB ? bfull : full;
            uint64_t* const rempty = TK_STREAM_SPLITB ? bempty : empty;
            uint32_t sb0 = smem_u32(sB), full0 = smem_u32(rfull), afull0 = smem_u32(afull), dempty0 = smem_u32(dempty);
            asm volatile("" : "+r"(sb0), "+r"(full0), "+r"(afull0), "+r"(dempty0));
            for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
                for (int k0 = 0; k0 < nk; k0 += kChunk, ++ch) {
                    const int b = ND == 2 ? (ch & 1) : 0;
                    if (ch >= ND) {  // this buffer's previous chunk has been added into the registers
                        bar_wait(dempty0 + b * 8, (ND == 2 ? (ch >> 1) - 1 : ch - 1) & 1);
                        __syncwarp();
                        sfence_after();
                    }
                    const int k1 = min(nk, k0 + kChunk);
                    for (int kc = k0; kc < k1; ++kc) {
                        bar_wait(full0 + s * 8, ph);  // (split rings: the factor ring's barriers)
                        const uint32_t bs = sb0 + s * C::STAGE_B;
                        bar_wait(afull0 + a * 8, aph);
                        __syncwarp();
                        sfence_after();
                        const uint32_t abuf = tm + uint32_t(C::A_BASE + a * MT * 32);
#pragma unroll
                        for (int ks = 0; ks < 2; ++ks) {
                            const uint64_t bd = sdesc(bs + ks * (64 * NH), 128, 256, 0);
#pragma unroll
                            for (int j = 0; j < MT; ++j) {
                                const uint32_t dm = tm + uint32_t((b * MT + j) * C::DW);
                                const uint32_t ahi = abuf + j * 32 + ks * 8;
                                mma_ts(dm, ahi, bd, id_main, (kc > k0 || ks > 0) ? 1u : 0u);
                                mma_ts(dm + NH, ahi + 16, bd, id_cross, 1u);
                            }
                        }
                        commit(&aempty[a]);
                        commit(&rempty[s]);
                        if (++s == RS) s = 0, ph ^= 1;
                        if (++a == NA) a = 0, aph ^= 1;
                    }
                    commit(&dfull[b]);
                }
            }
        }
    } else {
        // ===== converters (warps 0-7) =====
        const int quarter = warp & 3, khalf = warp >> 2;  // khalf: this warp's k share of a stage (0 .. kKSplit - 1)
        const int L = quarter * 32 + lane;  // TMEM lane
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        constexpr int ACC = C::ACC;
        const int c0 = khalf * (NH / kKSplit);  // this warp's accumulator columns
        uint32_t sy0 = smem_u32(sY), full0 = smem_u32(full), empty0 = smem_u32(empty), afull0 = smem_u32(afull),
                 aempty0 = smem_u32(aempty), dfull0 = smem_u32(dfull), dempty0 = smem_u32(dempty);
        asm volatile("" : "+r"(sy0), "+r"(full0), "+r"(empty0), "+r"(afull0), "+r"(aempty0), "+r"(dfull0), "+r"(dempty0));
        float acc[MT][ACC];
#pragma unroll
        for (int j = 0; j < MT; ++j)
#pragma unroll
            for (int e = 0; e < ACC; ++e) acc[j][e] = 0.f;
        int s = 0, a = 0;
        uint32_t ph = 0, aph = 0, ch = 0;
        // flush of chunk `pend` (buffer pend & 1) deferred by kDefer stages (past the converters'
        // lead over the MMA issuer), so the wait for its last MMAs does not stall the pipeline
        bool pending = false;
        int since = 0;
        // One buffer: flushed at once, the MMAs of the next chunk wait for it. (-DTK_STREAM_DEFER1=1:
        // the converters first fill the A ring with the next chunk's first NA - 1 stages, whose
        // buffers this chunk's MMAs release; measured 5-10 % slower.)
        constexpr int kDefer = ND == 2 ? NA + 2 : ((TK_STREAM_DEFER1 && NA >= 2) ? NA - 1 : 0);
        uint32_t pend = 0;
        auto flush = [&](uint32_t c) {
            const int b = ND == 2 ? (c & 1) : 0;
            bar_wait(dfull0 + b * 8, (ND == 2 ? (c >> 1) : c) & 1);
            sfence_after();
#pragma unroll
            for (int j = 0; j < MT; ++j) {
                const uint32_t base = tmem + lane_off + uint32_t((b * MT + j) * C::DW + c0);
#pragma unroll
                for (int cc = 0; cc < ACC; cc += 8) {
                    float m[8], x[8];
                    if (cc + 8 <= ACC) {
                        ld8(base + cc, m);
                        ld8(base + NH + cc, x);
                    } else if (cc + 4 <= ACC) {
                        ld4(base + cc, m);
                        ld4(base + NH + cc, x);
                        if (cc + 6 <= ACC) {
                            ld2(base + cc + 4, m + 4);
                            ld2(base + NH + cc + 4, x + 4);
                        }
                    } else {
                        ld2(base + cc, m);
                        ld2(base + NH + cc, x);
                    }
                    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        if (cc + e < ACC) acc[j][cc + e] += m[e] + x[e];
                }
            }
            sfence_before();
            __syncwarp();
            if (lane == 0) bar_arrive(dempty0 + b * 8);
        };
        const auto row_of = [&](int j) { return KM ? 128 * j + L : MT * L + j; };
        // M-major tiles of two q (bq = 2, MT = 2): rows [0, 128) of the tile are 128 p of q, rows
        // [128, 256) the same p of q + 1 (a thread's two adjacent rows share their q)
        const int BP = BM / bq;                       // p extent of a tile
        const int qo = (!KM && bq == 2 && L >= 64) ? 1 : 0;
        float* obase = nullptr;  // output tile of the pending last chunk
        int orows = 0, oq = 1;
        int64_t ostride = 0;
        bool store_after = false;
        const auto store = [&]() {
#pragma unroll
            for (int j = 0; j < MT; ++j) {
                const int row = row_of(j) - qo * BP;
                if (row < orows && qo < oq) {
                    // the address arithmetic stays here: without the barrier the compiler hoists
                    // the ACC store addresses into the k loop (recomputed every stage)
                    float* o = obase + row + int64_t(c0) * ostride + (qo ? ostride * cols : 0);
                    int64_t os = ostride;
                    asm volatile("" : "+l"(o), "+l"(os));
                    if (accum) {  // a K range of a split pass: add to the earlier ranges' sums
                        float prev[ACC];
#pragma unroll
                        for (int e = 0; e < ACC; ++e) prev[e] = (c0 + e < cols) ? o[e * os] : 0.f;
#pragma unroll
                        for (int e = 0; e < ACC; ++e) acc[j][e] += prev[e];
                    }
#pragma unroll
                    for (int e = 0; e < ACC; ++e)
                        if (c0 + e < cols) o[e * os] = acc[j][e];
                }
#pragma unroll
                for (int e = 0; e < ACC; ++e) acc[j][e] = 0.f;
            }
            store_after = false;
        };
        // raw Y values of one stage: this thread's MT rows x 8 k (its k half)
        float raw[MT][kKPW];
        const auto load_stage = [&](int st) {
            const uint32_t stage = sy0 + st * C::STAGE_Y;
            if constexpr (KM) {
                // row: 64 B with 16-B chunks at chunk ^ ((row >> 1) & 3) (64B swizzle)
#pragma unroll
                for (int j = 0; j < MT; ++j) {
                    const int row = 128 * j + L;
                    const uint32_t rb = stage + row * 64;
#pragma unroll
                    for (int h = 0; h < kKPW / 4; ++h) {
                        const int phys = ((kKPW / 4) * khalf + h) ^ ((row >> 1) & 3);
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n"
                                     : "=f"(raw[j][h * 4 + 0]), "=f"(raw[j][h * 4 + 1]), "=f"(raw[j][h * 4 + 2]),
                                       "=f"(raw[j][h * 4 + 3])
                                     : "r"(rb + phys * 16));
                    }
                }
            } else {
                // one box of 16 k-rows x BM p (4 BM bytes each, unswizzled): per k a warp
                // reads 32 MT consecutive p (conflict-free)
                // (two-q tiles: the box is [q][k][p] with BP p per row; the row stride stays a
                // compile-time immediate of the loads on either branch)
                const auto ld_rows = [&](auto bp_c, uint32_t bb) {
                    constexpr int kBP = decltype(bp_c)::value;
#pragma unroll
                    for (int kk = 0; kk < kKPW; ++kk) {
                        if constexpr (MT == 2) {
                            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];\n"
                                         : "=f"(raw[0][kk]), "=f"(raw[1][kk])
                                         : "r"(bb + kk * (kBP * 4)));
                        } else {
                            asm volatile("ld.shared.f32 %0, [%1];\n" : "=f"(raw[0][kk]) : "r"(bb + kk * (kBP * 4)));
                        }
                    }
                };
                if (bq == 2)
                    ld_rows(std::integral_constant<int, BM / 2>{},
                            stage + qo * (kSBK * (BM / 2) * 4) + khalf * kKPW * ((BM / 2) * 4) + (L * MT - qo * (BM / 2)) * 4);
                else
                    ld_rows(std::integral_constant<int, BM>{}, stage + khalf * kKPW * (BM * 4) + L * (MT * 4));
            }
        };
        for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int64_t q = (t / tiles_p) * bq;
            const int64_t p0 = (t % tiles_p) * BP;
            for (int kc = 0; kc < nk; ++kc) {
                bar_wait(full0 + s * 8, ph);
                load_stage(s);
                uint32_t hi[MT][kKPW], lo[MT][kKPW];
#pragma unroll
                for (int j = 0; j < MT; ++j)
#pragma unroll
                    for (int e = 0; e < kKPW; ++e) {
                        if constexpr (TR) split_hi_lo_trunc(raw[j][e], hi[j][e], lo[j][e]);
                        else if constexpr (TK_STREAM_PIPEBAL == 0) split_hi_lo(raw[j][e], hi[j][e], lo[j][e]);
                        else if (TK_STREAM_PIPEBAL == 1 && (e & 3) == 3) split_hi_lo_alu(raw[j][e], hi[j][e], lo[j][e]);
                        else split_hi_lo_fma(raw[j][e], one, hi[j][e], lo[j][e]);
                    }
                __syncwarp();
                if (lane == 0) bar_arrive(empty0 + s * 8);  // this warp's reads of the Y stage are done
                if (++s == ST) s = 0, ph ^= 1;
                bar_wait(aempty0 + a * 8, aph ^ 1);
                sfence_after();
                const uint32_t abuf = tmem + lane_off + uint32_t(C::A_BASE + a * MT * 32 + khalf * kKPW);
                if constexpr (kKPW == 16) {
#pragma unroll
                    for (int j = 0; j < MT; ++j) {
                        st16(abuf + j * 32, hi[j]);
                        st16(abuf + j * 32 + 16, lo[j]);
                    }
                } else if constexpr (kKPW == 8) {
                    if constexpr (MT == 2) st8_quad(abuf, hi[0], lo[0], hi[1], lo[1]);
                    else st8_pair(abuf, hi[0], lo[0]);
                } else {
                    if constexpr (MT == 2) st4_quad(abuf, hi[0], lo[0], hi[1], lo[1]);
                    else st4_pair(abuf, hi[0], lo[0]);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
                sfence_before();
                __syncwarp();
                if (lane == 0) bar_arrive(afull0 + a * 8);
                if (++a == NA) a = 0, aph ^= 1;
                // the previous chunk is added once the MMA issuer (up to NA stages behind the
                // converters) has certainly finished it: kDefer stages after its end
                if (pending && ++since >= kDefer) {
                    flush(pend);
                    pending = false;
                    if (store_after) store();  // the previous tile's last chunk: its rows are complete
                }
                if ((kc + 1) % kChunk == 0 || kc + 1 == nk) {
                    if (pending) {  // a short chunk: the older one first
                        flush(pend);
                        if (store_after) store();
                    }
                    pending = true;
                    since = 0;
                    pend = ch++;
                    if (kc + 1 == nk) {  // tile end: store once this chunk is flushed
                        store_after = true;
                        obase = out + q * P * cols + p0;
                        orows = static_cast<int>(lmin(BP, P - p0));
                        oq = static_cast<int>(lmin(bq, Q - q));
                        ostride = P;
                    }
                    if constexpr (kDefer == 0) {
                        flush(pend);
                        pending = false;
                        if (store_after) store();
                    }
                }
            }
            if (t + gridDim.x >= ntiles && pending) {  // last tile of this CTA: flush and store now
                flush(pend);
                pending = false;
                store();
            }
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

template <int NH, bool KM, int MT, int OCC, int CH, bool TR>
void launch_stream_ch(const float* in, const uint8_t* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                      cudaStream_t s, bool accum) {
    using C = SCfg<NH, KM, MT, OCC>;
    static bool attr = false;
    if (!attr) {
        TK_CUDA(cudaFuncSetAttribute(ttm_stream_kernel<NH, KM, MT, OCC, CH, TR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(C::smem)));
        attr = true;
    }
    require(K < (int64_t(1) << 31) && Q < (int64_t(1) << 31) && P < (int64_t(1) << 31), "ttm: extent too large for TMA");
    CUtensorMap map;
    CUresult r;
    int64_t tiles_p, ntiles, rows, qext = 1;
    int bq = 1;
    if constexpr (KM) {  // Q rows of K contiguous values
        tiles_p = (Q + C::BM - 1) / C::BM;
        ntiles = tiles_p;
        rows = Q;
        const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(Q)};
        const cuuint64_t strides[1] = {cuuint64_t(K) * 4};
        const cuuint32_t box[2] = {kSBK, C::BOXR};
        const cuuint32_t estr[2] = {1, 1};
        r = encode_tiled2()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(in), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        // tiles of BM p of one q, or (MT = 2) of BM / 2 p of two q where that wastes fewer of the
        // tile's rows on the ragged end of P (2400 = 9.4 x 256 = 18.75 x 128: 6.3% -> 1.3% idle rows)
        static const bool no_bq = [] {
            const char* e = std::getenv("TENKIT_STREAM_BQ");
            return e && e[0] == '1';
        }();
        if (MT == 2 && !no_bq && Q >= 2) {
            const double w1 = double((P + C::BM - 1) / C::BM * C::BM) / double(P);
            const double w2 = double((P + C::BM / 2 - 1) / (C::BM / 2) * (C::BM / 2)) / double(P) * double((Q + 1) / 2 * 2) / double(Q);
            if (w2 < w1 - 0.005) bq = 2;
        }
        const int bp = C::BM / bq;
        tiles_p = (P + bp - 1) / bp;
        ntiles = tiles_p * ((Q + bq - 1) / bq);
        rows = P;
        qext = Q;
        const cuuint64_t dims[3] = {cuuint64_t(P), cuuint64_t(K), cuuint64_t(Q)};
        const cuuint64_t strides[2] = {cuuint64_t(P) * 4, cuuint64_t(P) * cuuint64_t(K) * 4};
        const cuuint32_t box[3] = {cuuint32_t(bp), kSBK, cuuint32_t(bq)};
        const cuuint32_t estr[3] = {1, 1, 1};
        r = encode_tiled2()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    const int64_t grid = std::min<int64_t>(ntiles, int64_t(C::OCC) * 148);
    TK_MAXSMEM((ttm_stream_kernel<NH, KM, MT, OCC, CH, TR>));
    ttm_stream_kernel<NH, KM, MT, OCC, CH, TR><<<static_cast<unsigned>(grid), kSThreads, C::smem, s>>>(map, bpk, out, rows, K,
                                                                                             cols, tiles_p, ntiles,
                                                                                             accum ? 1 : 0, bq, qext, 1u);
    TK_LAUNCH_CHECK();
}

// Two 128-row M tiles per CTA, one CTA per SM: the per-stage barrier and address work of the
// converters, the factor k-block and the MMA issue are shared by both tiles (measured: 0.79 of
// the HBM peak at cfg3 against 0.71 with one tile per CTA and two CTAs per SM; NH = 64, whose
// two tiles leave TMEM room for one accumulator buffer only: 0.76 against 0.63). A/B knobs:
// TENKIT_STREAM_MT=1 (one tile per CTA, two CTAs per SM), TENKIT_STREAM_BQ=1 (M-major tiles
// never span two q).
template <int NH, bool KM, int MT, int OCC>
void launch_stream_mt(const float* in, const uint8_t* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                      cudaStream_t s, bool accum) {
    static const bool tr = [] {
        const char* e = std::getenv("TENKIT_STREAM_TRUNC");
        return e && e[0] == '1';
    }();
    if (tr) launch_stream_ch<NH, KM, MT, OCC, kChunkDefault, true>(in, bpk, out, P, K, Q, cols, s, accum);
    else launch_stream_ch<NH, KM, MT, OCC, kChunkDefault, false>(in, bpk, out, P, K, Q, cols, s, accum);
}

template <int NH, bool KM>
void launch_stream(const float* in, const uint8_t* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                   cudaStream_t s, bool accum) {
    static const int mt = [] {
        const char* e = std::getenv("TENKIT_STREAM_MT");
        return e ? std::atoi(e) : 0;
    }();
    const int m = mt == 1 ? 1 : 2;
    if (m == 2) launch_stream_mt<NH, KM, 2, 1>(in, bpk, out, P, K, Q, cols, s, accum);
    else launch_stream_mt<NH, KM, 1, 2>(in, bpk, out, P, K, Q, cols, s, accum);
}

// NH = cols rounded up to 8 (A/B knob TENKIT_STREAM_NH16=1: to 16, the first design's padding)
inline int stream_nh(int cols) {
    static const bool r16 = [] {
        const char* e = std::getenv("TENKIT_STREAM_NH16");
        return e && e[0] == '1';
    }();
    return std::max(16, r16 ? (cols + 15) / 16 * 16 : (cols + 7) / 8 * 8);
}

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
    if (cols < 1 || cols > kMaxRank || K < kSBK) return false;
    if (P == 1) return K % 4 == 0 && (Q + 255) / 256 >= 148;  // K-major: >= one wave of 2 x 128-row tiles
    return P % 4 == 0 && P >= 256 && (P + 255) / 256 * Q >= 2 * 148;
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

int64_t stream_pack_kblock_bytes(int cols) { return 128 * int64_t(stream_nh(cols)); }

// P == 1: contraction over mode 0, transposed output out[q + r Q]; else out[p + r P + q P cols].
// k0 (a multiple of 16) / accumulate: the pass covers rows [k0, k0 + K) of the packed factor and
// adds to `out` (one K range of a pass split over K; `in` points at the range's first k).
void launch_ttm_stream(const float* in, const void* bpk, float* out, int64_t P, int64_t K, int64_t Q, int cols,
                       cudaStream_t s, int64_t k0, bool accum) {
    require(k0 % kSBK == 0, "ttm: split ranges start at multiples of 16");
    const int nh = stream_nh(cols);
    const uint8_t* b = static_cast<const uint8_t*>(bpk) + (k0 / kSBK) * stream_pack_kblock_bytes(cols);
#define TK_STREAM_CASE(N)                                                   \
    case N:                                                                 \
        if (P == 1) launch_stream<N, true>(in, b, out, P, K, Q, cols, s, accum);   \
        else launch_stream<N, false>(in, b, out, P, K, Q, cols, s, accum);         \
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
