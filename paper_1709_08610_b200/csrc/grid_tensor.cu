// grid_tensor.cu -- K1t: Eq. (2) for SLOPE2 and SLOPE3 (one GEMM per z0 value) as a dense
// contraction on the 5th-generation tensor cores (tcgen05.mma, accumulators in TMEM).
//
// Same exact factorisation as K1s (grid_separable.cu):
//     R[i][j] = sum_k EX[i][k] * EY[j][k],  EX = 2^(-K (x - tx z)^2),  EY = 2^(-K (y - ty z)^2).
// fp32 accuracy on TF32 tensor cores by the 3xTF32 split: every factor v is written as
// v = hi + lo with hi = v truncated to TF32 (exact) and lo = v - hi (exact in fp32, then seen
// with TF32's 11 significant bits), and the K dimension is concatenated three times,
//     [EX_hi | EX_hi | EX_lo] . [EY_hi | EY_lo | EY_hi]^T,
// so one accumulator receives hi.hi + hi.lo + lo.hi (the dropped lo.lo term is ~2^-22 relative).
// All terms are positive (no cancellation), so the relative error of R stays ~1e-6 (T1).
//
// CTA = 256 threads, one 128 (tx) x 256 (ty) output tile of one event, 1 CTA per SM (~200 KB
// smem).  Hits are staged once in shared memory by TMA bulk copies (HitStage).  Per 32-hit
// chunk all 8 warps GENERATE the split operands (one MUFU.EX2 per factor) into one of two
// operand stages (K-major, no-swizzle UMMA canonical layout), then thread 0 issues
// 4 k-steps x 3 parts = 12 tcgen05.mma (M=128, N=256, K=8, kind::tf32) and commits them to the
// stage's mbarrier; the next chunk is generated into the other stage while the tensor core
// works.  Epilogue: tcgen05.ld (32x32b.x16) TMEM -> registers -> coalesced-by-row stores.
#include "common.cuh"
#include "kernels.cuh"
#include "tcgen05.cuh"

#include <cuda_fp16.h>

namespace retina {

#ifndef RETINA_TC_KC
#define RETINA_TC_KC 32
#endif
#ifndef RETINA_TC_MINB
#define RETINA_TC_MINB 1
#endif
constexpr int TC_KC = RETINA_TC_KC;  // hits per chunk (tile TC_M x TC_N in tcgen05.cuh)
constexpr int TC_A_BYTES = TC_M * TC_KC * 4;             // one part (hi or lo) of A: 16 KB
constexpr int TC_B_BYTES = TC_N * TC_KC * 4;             // one part of B: 32 KB
constexpr int TC_STAGE_BYTES = 2 * TC_A_BYTES + 2 * TC_B_BYTES;  // 96 KB
constexpr int TC_TMEM_COLS = 256;
#ifndef RETINA_TC_WARPS
#define RETINA_TC_WARPS 16
#endif
constexpr int TC_WARPS = RETINA_TC_WARPS;  // 8 or 16: warps per CTA (all generate operands)
constexpr int TC_KB = TC_KC / 4;           // 4-hit k-blocks per chunk
constexpr int TC_NR = TC_WARPS / TC_KB;    // row sets per k-block
static_assert(TC_WARPS == 8 || TC_WARPS == 16, "8 or 16 warps");
static_assert(TC_NR >= 1 && 4 % TC_NR == 0, "warps / k-blocks must divide the 4 A row groups");

// Epilogue shared by the tensor-core grid kernels: warp w reads TMEM lanes 32 (w % 4) .. +31
// (= tile rows) and column group w / 4 of the 128 x 256 fp32 accumulator, and stores them.
// SPLIT16: the fp16-split kernel keeps two accumulators, D1 = sum hi.hi (scaled 2^30) in columns
// [0, 256) and D2 = sum (hi.lo + lo.hi) (scaled 2^41) in [256, 512); R = D1 2^-30 + D2 2^-41.
template <int MODEL, bool SPLIT16 = false>
__device__ __forceinline__ void tc_epilogue(const GridArgs &a, int e, int t_m, int t_n, int l, int nl, uint32_t tmem,
                                            int n_chunks, int warp, int lane) {
    constexpr int GROUP_COLS = TC_N / (TC_WARPS / 4);
    const int q = warp & 3, half = warp >> 2;
    const int i = t_m * TC_M + q * 32 + lane;
    const int64_t cells = (int64_t)a.n0 * a.n1 * nl;
    float *out = a.R + (int64_t)e * cells + ((int64_t)l * a.n0 + i) * a.n1;  // z0 plane l (Z37)
#pragma unroll 1
    for (int cc = 0; cc < GROUP_COLS / 16; ++cc) {
        const int col = half * GROUP_COLS + cc * 16;
        uint32_t v[16];
        if (n_chunks > 0) {
            const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)col;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                  "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                  "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            if constexpr (SPLIT16) {
                uint32_t u[16];
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                    "[%16];"
                    : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]),
                      "=r"(u[7]), "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]),
                      "=r"(u[14]), "=r"(u[15])
                    : "r"(taddr + (uint32_t)TC_N));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int x = 0; x < 16; ++x)
                    v[x] = __float_as_uint(__fmaf_rn(__uint_as_float(u[x]), 0x1p-41f,
                                                     __fmul_rn(__uint_as_float(v[x]), 0x1p-30f)));
            } else {
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            }
        } else {
#pragma unroll
            for (int x = 0; x < 16; ++x) v[x] = 0u;
        }
        const int j0 = t_n * TC_N + col;
        if (i < a.n0) {
            if (j0 + 15 < a.n1 && (((uintptr_t)(out + j0)) & 15u) == 0) {
#pragma unroll
                for (int x = 0; x < 16; x += 4)
                    *reinterpret_cast<float4 *>(out + j0 + x) =
                        make_float4(__uint_as_float(v[x]), __uint_as_float(v[x + 1]), __uint_as_float(v[x + 2]),
                                    __uint_as_float(v[x + 3]));
            } else {
#pragma unroll
                for (int x = 0; x < 16; ++x)
                    if (j0 + x < a.n1) out[j0 + x] = __uint_as_float(v[x]);
            }
        }
    }
}

template <int MODEL, bool ZREF>
__global__ void __launch_bounds__(32 * TC_WARPS, RETINA_TC_MINB) grid_tensor_kernel(GridArgs a) {
    extern __shared__ __align__(1024) uint8_t s_raw[];
    __shared__ __align__(8) uint64_t s_bar[2];     // hit stage
    __shared__ __align__(8) uint64_t s_empty[2];   // operand stage s free (MMAs done)
    __shared__ uint32_t s_tmem;

    uint8_t *stage_base = s_raw;                                           // 2 x 96 KB operands
    float4 *s_hits = reinterpret_cast<float4 *>(s_raw + 2 * TC_STAGE_BYTES);  // hit stage after

    const int e = a.e_base + blockIdx.y;
    // block order: z0 index fastest (SLOPE3); each block writes row segments of its z0 plane
    const int tn = (a.n1 + TC_N - 1) / TC_N;
    const int nl = (MODEL == kSlope3) ? a.n2 : 1;
    const int l = blockIdx.x % nl, tile = blockIdx.x / nl;
    const int t_n = tile % tn, t_m = tile / tn;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (warp == 0) {  // TMEM accumulator: 128 lanes x 256 fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(TC_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        tc_fence_before();
    }
    if (tid == 0) {
        mbar_init(&s_empty[0], 1);
        mbar_init(&s_empty[1], 1);
    }
    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;
    HitStage st;
    st.init(s_hits, s_bar, a.hits + start, nh, a.cap);  // contains __syncthreads (+ mbarrier fence)
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    // generation roles: warp % TC_KB = k-block (4 hits) of the chunk; operand rows
    // lane + 32 (t TC_NR + warp / TC_KB): 4 / TC_NR rows of A and 8 / TC_NR rows of B per thread
    const int kb = warp % TC_KB, rset = warp / TC_KB;
    constexpr int NA = 4 / TC_NR, NB = 8 / TC_NR;
    float pa[NA], pb[NB];
#pragma unroll
    for (int t = 0; t < NA; ++t)
        pa[t] = __ldg(a.nodes0 + min(t_m * TC_M + lane + 32 * (t * TC_NR + rset), a.n0 - 1));
#pragma unroll
    for (int t = 0; t < NB; ++t)
        pb[t] = __ldg(a.nodes1 + min(t_n * TC_N + lane + 32 * (t * TC_NR + rset), a.n1 - 1));
    const float negK = a.negK;
    const float zref = (MODEL == kSlope3) ? __ldg(a.nodes2 + l) : a.z_ref;  // d = z - z0 or z - z_ref
    const uint32_t stage_saddr = smem_u32(stage_base);

    int chunk = 0;  // global chunk counter (uniform)
    st.pass([&](const float4 *h, int len) {
        for (int k0 = 0; k0 < len; k0 += TC_KC, ++chunk) {
            const int s = chunk & 1;
            if (chunk >= 2) mbar_wait(&s_empty[s], ((chunk - 2) >> 1) & 1);  // MMAs of chunk-2 done
            uint8_t *sb = stage_base + s * TC_STAGE_BYTES;
            // ---- generate this warp's k-block (4 hits) for 4 A rows and 8 B rows per lane
            float hx[4], hy[4], hz[4], hzl[4];
            bool ok[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = k0 + kb * 4 + q;
                ok[q] = k < len;
                const float4 hk = h[ok[q] ? k : 0];
                hx[q] = hk.x;
                hy[q] = hk.y;
                if (ZREF || MODEL == kSlope3)
                    two_sum(hk.z, -zref, hz[q], hzl[q]);
                else {
                    hz[q] = hk.z;
                    hzl[q] = 0.f;
                }
            }
            float *Ahi = reinterpret_cast<float *>(sb);
            float *Alo = reinterpret_cast<float *>(sb + TC_A_BYTES);
            float *Bhi = reinterpret_cast<float *>(sb + 2 * TC_A_BYTES);
            float *Blo = reinterpret_cast<float *>(sb + 2 * TC_A_BYTES + TC_B_BYTES);
#pragma unroll
            for (int t = 0; t < NA + NB; ++t) {
                const bool isA = t < NA;
                const float p = isA ? pa[t] : pb[t - NA];
                float vh[4], vl[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float c = isA ? hx[q] : hy[q];
                    const float sres = (ZREF || MODEL == kSlope3) ? __fmaf_rn(-p, hzl[q], __fmaf_rn(-p, hz[q], c))
                                                                   : __fmaf_rn(-p, hz[q], c);
                    const float v = ok[q] ? ex2_approx(__fmul_rn(__fmul_rn(sres, sres), negK)) : 0.f;
                    vh[q] = tf32_trunc(v);
                    vl[q] = __fsub_rn(v, vh[q]);
                }
                // K-major no-swizzle canonical layout: k-block kb of 4 elements, row r at 16 B
                const int r = lane + 32 * ((isA ? t : t - NA) * TC_NR + rset);
                const int rows = isA ? TC_M : TC_N;
                float *dh = (isA ? Ahi : Bhi) + (kb * rows + r) * 4;
                float *dl = (isA ? Alo : Blo) + (kb * rows + r) * 4;
                *reinterpret_cast<float4 *>(dh) = make_float4(vh[0], vh[1], vh[2], vh[3]);
                *reinterpret_cast<float4 *>(dl) = make_float4(vl[0], vl[1], vl[2], vl[3]);
            }
            fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
            __syncthreads();
            if (tid == 0) {
                tc_fence_after();
                const uint32_t base = stage_saddr + s * TC_STAGE_BYTES;
                const uint32_t aH = base, aL = base + TC_A_BYTES, bH = base + 2 * TC_A_BYTES,
                               bL = bH + TC_B_BYTES;
#pragma unroll
                for (int j = 0; j < TC_KC / 8; ++j) {  // K = 8 tf32 per MMA = 2 k-blocks
                    const uint32_t oa = j * 2 * (TC_M * 16), ob = j * 2 * (TC_N * 16);
                    const uint32_t acc0 = (chunk > 0 || j > 0) ? 1u : 0u;
                    // LBO = distance between the two 4-element k-blocks, SBO = 8 rows x 16 B
                    tc_mma(tmem, umma_desc(aH + oa, TC_M * 16, 128), umma_desc(bH + ob, TC_N * 16, 128), acc0);
                    tc_mma(tmem, umma_desc(aH + oa, TC_M * 16, 128), umma_desc(bL + ob, TC_N * 16, 128), 1u);
                    tc_mma(tmem, umma_desc(aL + oa, TC_M * 16, 128), umma_desc(bH + ob, TC_N * 16, 128), 1u);
                }
                tc_commit(&s_empty[s]);
            }
        }
    });

    const int n_chunks = chunk;
    if (n_chunks > 0) {
        const int s = (n_chunks - 1) & 1;
        mbar_wait(&s_empty[s], ((n_chunks - 1) >> 1) & 1);  // last MMAs (and all before) done
    }
    tc_fence_after();

    tc_epilogue<MODEL>(a, e, t_m, t_n, l, nl, tmem, n_chunks, warp, lane);
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS));
}


// ------------------------------------------------------------------------------------------------
// F16 split variant (RETINA_GRID_TENSOR_F16): the same contraction with fp16 operands on
// kind::f16 (twice the tf32 rate per MMA byte).  Each factor v in [0, 1] is split exactly as
//     v = hi 2^-15 + lo,   hi = fp16_rn(v 2^15) (11 significant bits, exact back in fp32),
//     lo = v - hi 2^-15 (exact in fp32, |lo| <= 2^-12 v), stored as fp16_rn(lo 2^26);
// two TMEM accumulators take D1 = sum hi_x hi_y (scale 2^30) and D2 = sum (hi_x lo_y + lo_x hi_y)
// (scale 2^41), and the epilogue forms R = D1 2^-30 + D2 2^-41.  Per term the error is the dropped
// lo.lo (<= 2^-24 relative) plus the fp16 rounding of lo (<= 2^-24 relative); the scales keep
// hi normal down to v = 2^-29 and lo normal down to 2^-40 (below that, absolute errors
// < 2^-50), so the result meets the same T1 budget as the 3xTF32 kernel with half the MMAs.
// CTA = 16 generating warps + 1 MMA warp, one 128 x 256 tile.  Per chunk of T16_KC hits each
// generating warp writes one 8-hit k-block (16 B of fp16 per row and part) for NA A rows and NB B
// rows per lane into stage c % T16_NS, then arrives on full[stage]; the MMA warp waits full, issues
// the chunk's MMAs and commits them to empty[stage], which the generating warps wait on before
// refilling it.  No block-wide barrier per chunk: warps run ahead as far as the ring allows.
#ifndef RETINA_T16_KC
#define RETINA_T16_KC 64
#endif
#ifndef RETINA_T16_NS
#define RETINA_T16_NS 2
#endif
constexpr int T16_KC = RETINA_T16_KC;               // hits per chunk
constexpr int T16_NS = RETINA_T16_NS;               // operand stages in the ring
constexpr int T16_KB = T16_KC / 8;                  // 8-hit k-blocks per chunk
constexpr int T16_A_BYTES = TC_M * T16_KC * 2;      // one part (hi or lo) of A: fp16
constexpr int T16_B_BYTES = TC_N * T16_KC * 2;
constexpr int T16_STAGE_BYTES = 2 * T16_A_BYTES + 2 * T16_B_BYTES;
constexpr int T16_WARPS = 16;                       // generating warps (+1 MMA warp)
constexpr int T16_NR = T16_WARPS / T16_KB;          // row sets per k-block
static_assert(T16_NR >= 1 && 4 % T16_NR == 0, "warps / k-blocks must divide the 4 A row groups");
static_assert(T16_KC % 16 == 0, "K = 16 per kind::f16 MMA");
static_assert(T16_NS * T16_STAGE_BYTES + 1024 + 64 * 16 <= 227 * 1024, "operand ring must leave room for hits");

template <int MODEL, bool ZREF>
__global__ void __launch_bounds__(32 * (T16_WARPS + 1), 1) grid_tensor16_kernel(GridArgs a) {
    extern __shared__ __align__(1024) uint8_t s_raw[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ __align__(8) uint64_t s_full[T16_NS];
    __shared__ __align__(8) uint64_t s_empty[T16_NS];
    __shared__ __align__(8) uint64_t s_done;
    __shared__ uint32_t s_tmem;

    uint8_t *stage_base = s_raw;
    float4 *s_hits = reinterpret_cast<float4 *>(s_raw + T16_NS * T16_STAGE_BYTES);

    const int e = a.e_base + blockIdx.y;
    const int tn = (a.n1 + TC_N - 1) / TC_N;
    const int nl = (MODEL == kSlope3) ? a.n2 : 1;
    const int l = blockIdx.x % nl, tile = blockIdx.x / nl;
    const int t_n = tile % tn, t_m = tile / tn;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool mma_warp = warp == T16_WARPS;

    if (warp == 0) {  // two accumulators: 128 lanes x (256 + 256) fp32 columns = all of TMEM
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(2 * TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        tc_fence_before();
    }
    if (tid == 0) {
        for (int i = 0; i < T16_NS; ++i) {
            mbar_init(&s_full[i], T16_WARPS);
            mbar_init(&s_empty[i], 1);
        }
        mbar_init(&s_done, 1);
    }
    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;
    HitStage st;
    st.init(s_hits, s_bar, a.hits + start, nh, a.cap);  // __syncthreads: barrier inits visible
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    const int kb = warp % T16_KB, rset = (warp / T16_KB) % T16_NR;
    constexpr int NA = 4 / T16_NR, NB = 8 / T16_NR;
    float pa[NA], pb[NB];
    if (!mma_warp) {
#pragma unroll
        for (int t = 0; t < NA; ++t)
            pa[t] = __ldg(a.nodes0 + min(t_m * TC_M + lane + 32 * (t * T16_NR + rset), a.n0 - 1));
#pragma unroll
        for (int t = 0; t < NB; ++t)
            pb[t] = __ldg(a.nodes1 + min(t_n * TC_N + lane + 32 * (t * T16_NR + rset), a.n1 - 1));
    }
    const float negK = a.negK;
    const float zref = (MODEL == kSlope3) ? __ldg(a.nodes2 + l) : a.z_ref;
    const uint32_t stage_saddr = smem_u32(stage_base);
    constexpr bool EXACT_D = ZREF || MODEL == kSlope3;

    int chunk = 0;
    st.pass([&](const float4 *h, int len) {
        for (int k0 = 0; k0 < len; k0 += T16_KC, ++chunk) {
            const int s = chunk % T16_NS;
            const uint32_t round = (uint32_t)(chunk / T16_NS);
            if (mma_warp) {
                if (lane == 0) {
                    mbar_wait(&s_full[s], round & 1u);
                    tc_fence_after();
                    const uint32_t base = stage_saddr + s * T16_STAGE_BYTES;
                    const uint32_t aH = base, aL = base + T16_A_BYTES, bH = base + 2 * T16_A_BYTES,
                                   bL = bH + T16_B_BYTES;
#pragma unroll
                    for (int j = 0; j < T16_KC / 16; ++j) {  // K = 16 fp16 per MMA = 2 k-blocks
                        const uint32_t oa = j * 2 * (TC_M * 16), ob = j * 2 * (TC_N * 16);
                        const uint32_t acc0 = (chunk > 0 || j > 0) ? 1u : 0u;
                        tc_mma_f16(tmem, umma_desc(aH + oa, TC_M * 16, 128), umma_desc(bH + ob, TC_N * 16, 128),
                                   acc0);
                        tc_mma_f16(tmem + TC_N, umma_desc(aH + oa, TC_M * 16, 128),
                                   umma_desc(bL + ob, TC_N * 16, 128), acc0);
                        tc_mma_f16(tmem + TC_N, umma_desc(aL + oa, TC_M * 16, 128),
                                   umma_desc(bH + ob, TC_N * 16, 128), 1u);
                    }
                    tc_commit(&s_empty[s]);
                }
                __syncwarp();
                continue;
            }
            if (chunk >= T16_NS) mbar_wait(&s_empty[s], (round - 1) & 1u);  // MMAs of chunk - NS done
            uint8_t *sb = stage_base + s * T16_STAGE_BYTES;
            // hits of this warp's k-block as pairs (q, q+1); a missing hit gets a huge coordinate
            // so its factor is exactly ex2(-inf) = 0 (no per-element select)
            float2 hx[4], hy[4], hz[4], hzl[4];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int k = k0 + kb * 8 + q;
                const bool ok = k < len;
                const float4 hk = h[ok ? k : 0];
                float zh = hk.z, zl = 0.f;
                if (EXACT_D) two_sum(hk.z, -zref, zh, zl);
                float *X = (q & 1) ? &hx[q >> 1].y : &hx[q >> 1].x;
                float *Y = (q & 1) ? &hy[q >> 1].y : &hy[q >> 1].x;
                float *Z = (q & 1) ? &hz[q >> 1].y : &hz[q >> 1].x;
                float *ZL = (q & 1) ? &hzl[q >> 1].y : &hzl[q >> 1].x;
                *X = ok ? hk.x : 1e30f;
                *Y = ok ? hk.y : 1e30f;
                *Z = zh;
                *ZL = zl;
            }
            const float2 nk2 = make_float2(negK, negK);
#pragma unroll
            for (int t = 0; t < NA + NB; ++t) {
                const bool isA = t < NA;
                const float p = isA ? pa[t] : pb[t - NA];
                const float2 mp = make_float2(-p, -p);
                uint32_t wh[4], wl[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 c = isA ? hx[q] : hy[q];
                    const float2 sres = EXACT_D ? __ffma2_rn(mp, hzl[q], __ffma2_rn(mp, hz[q], c)) : __ffma2_rn(mp, hz[q], c);
                    const float2 arg = __fmul2_rn(__fmul2_rn(sres, sres), nk2);
                    const float2 v = make_float2(ex2_approx(arg.x), ex2_approx(arg.y));
                    const float2 vs = __fmul2_rn(v, make_float2(0x1p15f, 0x1p15f));
                    const __half2 hh = __floats2half2_rn(vs.x, vs.y);
                    const float2 hf = __half22float2(hh);                             // exact
                    const float2 lo = __ffma2_rn(hf, make_float2(-0x1p-15f, -0x1p-15f), v);  // exact: v - hi 2^-15
                    const float2 ls = __fmul2_rn(lo, make_float2(0x1p26f, 0x1p26f));
                    wh[q] = *reinterpret_cast<const uint32_t *>(&hh);
                    wl[q] = pack_h2(ls.x, ls.y);
                }
                // K-major no-swizzle canonical layout: k-block kb of 8 fp16 elements, row r at 16 B
                const int r = lane + 32 * ((isA ? t : t - NA) * T16_NR + rset);
                const int rows = isA ? TC_M : TC_N;
                uint8_t *dh = sb + (isA ? 0 : 2 * T16_A_BYTES) + (size_t)(kb * rows + r) * 16;
                uint8_t *dl = dh + (isA ? T16_A_BYTES : T16_B_BYTES);
                *reinterpret_cast<uint4 *>(dh) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
                *reinterpret_cast<uint4 *>(dl) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
            }
            fence_proxy_async();  // this thread's generic-proxy stores -> visible to the tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_full[s]);
        }
    });

    const int n_chunks = chunk;
    if (mma_warp && lane == 0) {
        if (n_chunks > 0) tc_commit(&s_done);  // arrives once every MMA issued so far is complete
        else mbar_arrive(&s_done);
    }
    mbar_wait(&s_done, 0u);
    tc_fence_after();
    if (!mma_warp) tc_epilogue<MODEL, true>(a, e, t_m, t_n, l, nl, tmem, n_chunks, warp, lane);
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_N));
}

// ------------------------------------------------------------------------------------------------
// CTA-pair variant of the fp16-split kernel (cta_group::2): a cluster of two CTAs on one TPC
// computes a 256 (tx) x 256 (ty) tile with M = 256 MMAs issued by the even CTA.  CTA r holds
// the A rows (tx) 128 r .. 128 r + 127 of the pair tile and HALF of the B operand (ty rows
// 128 r .. 128 r + 127); its TMEM receives its own 128 rows x 256 columns.  Each CTA therefore
// generates 128 + 128 factor rows per hit for 32,768 pairs instead of 128 + 256: a third less
// generation work, which is what limits the one-CTA kernel.  The odd CTA's generating warps
// arrive on the even CTA's full barrier (mapa + mbarrier.arrive.release.cluster); the MMA
// commit is multicast to both CTAs' empty barriers.
#ifndef RETINA_X2_NS
#define RETINA_X2_NS 2
#endif
#ifndef RETINA_X2_KC
#define RETINA_X2_KC 64
#endif
constexpr int X2_KC = RETINA_X2_KC;                    // hits per chunk
constexpr int X2_NS = RETINA_X2_NS;
constexpr int X2_KB = X2_KC / 8;                       // 8-hit k-blocks per chunk
constexpr int X2_PART = 128 * X2_KC * 2;               // one fp16 part (hi or lo) of A or of B-half
constexpr int X2_STAGE = 4 * X2_PART;                  // A hi, A lo, B hi, B lo: 64 KB
constexpr int X2_WARPS = 16;                           // generating warps (+1 MMA warp)
constexpr int X2_NR = X2_WARPS / X2_KB;                // row sets per k-block (2)
constexpr int X2_NA = 4 / X2_NR, X2_NB = 4 / X2_NR;   // A and B rows per lane per chunk (2, 2)
static_assert(X2_NS * X2_STAGE + 1024 + 64 * 16 <= 227 * 1024, "operand ring must leave room for hits");

template <int MODEL, bool ZREF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (X2_WARPS + 1), 1)
    grid_tensor16x2_kernel(GridArgs a) {
    extern __shared__ __align__(1024) uint8_t s_raw[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ __align__(8) uint64_t s_full[X2_NS];   // used in the even CTA: 2 x 16 warps arrive
    __shared__ __align__(8) uint64_t s_empty[X2_NS];  // both CTAs: the multicast MMA commit arrives
    __shared__ __align__(8) uint64_t s_done;
    __shared__ uint32_t s_tmem;

    uint8_t *stage_base = s_raw;
    float4 *s_hits = reinterpret_cast<float4 *>(s_raw + X2_NS * X2_STAGE);

    const uint32_t rank = cluster_rank();
    const int e = a.e_base + blockIdx.y;
    const int tn = (a.n1 + TC_N - 1) / TC_N;
    const int nl = (MODEL == kSlope3) ? a.n2 : 1;
    const int pair = blockIdx.x >> 1;  // one pair tile per cluster
    const int l = pair % nl, tile = pair / nl;
    const int t_n = tile % tn, p_m = tile / tn;
    const int t_m = 2 * p_m + (int)rank;  // this CTA's 128-row block of tx
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const bool mma_warp = warp == X2_WARPS;

    if (warp == 0) {  // both CTAs: 2 accumulators (hi.hi and hi.lo + lo.hi) x 256 columns
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(2 * TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        tc_fence_before();
    }
    if (tid == 0) {
        for (int i = 0; i < X2_NS; ++i) {
            mbar_init(&s_full[i], 2 * X2_WARPS);
            mbar_init(&s_empty[i], 1);
        }
        mbar_init(&s_done, 1);
        fence_mbar_init();
    }
    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;
    HitStage st;
    st.init(s_hits, s_bar, a.hits + start, nh, a.cap);  // __syncthreads inside
    cluster_sync_all();                                 // peer barriers initialised before remote arrives
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    const int kb = warp % X2_KB, rset = (warp / X2_KB) % X2_NR;
    float pa[X2_NA], pb[X2_NB];
    if (!mma_warp) {
#pragma unroll
        for (int t = 0; t < X2_NA; ++t)
            pa[t] = __ldg(a.nodes0 + min(t_m * 128 + lane + 32 * (t * X2_NR + rset), a.n0 - 1));
#pragma unroll
        for (int t = 0; t < X2_NB; ++t)  // this CTA's half of the pair tile's 256 ty columns
            pb[t] = __ldg(a.nodes1 + min(t_n * TC_N + (int)rank * 128 + lane + 32 * (t * X2_NR + rset), a.n1 - 1));
    }
    const float negK = a.negK;
    const float zref = (MODEL == kSlope3) ? __ldg(a.nodes2 + l) : a.z_ref;
    const uint32_t stage_saddr = smem_u32(stage_base);
    constexpr bool EXACT_D = ZREF || MODEL == kSlope3;

    int chunk = 0;
    st.pass([&](const float4 *h, int len) {
        for (int k0 = 0; k0 < len; k0 += X2_KC, ++chunk) {
            const int s = chunk % X2_NS;
            const uint32_t round = (uint32_t)(chunk / X2_NS);
            if (mma_warp) {
                if (rank == 0 && lane == 0) {
                    mbar_wait_cluster(&s_full[s], round & 1u);
                    tc_fence_after();
                    const uint32_t base = stage_saddr + s * X2_STAGE;
                    const uint32_t aH = base, aL = base + X2_PART, bH = base + 2 * X2_PART, bL = base + 3 * X2_PART;
#pragma unroll
                    for (int j = 0; j < X2_KC / 16; ++j) {  // K = 16 fp16 per MMA = 2 k-blocks
                        const uint32_t o = j * 2 * (128 * 16);
                        const uint32_t acc0 = (chunk > 0 || j > 0) ? 1u : 0u;
                        tc2_mma_f16(tmem, umma_desc(aH + o, 128 * 16, 128), umma_desc(bH + o, 128 * 16, 128), acc0);
                        tc2_mma_f16(tmem + TC_N, umma_desc(aH + o, 128 * 16, 128), umma_desc(bL + o, 128 * 16, 128),
                                    acc0);
                        tc2_mma_f16(tmem + TC_N, umma_desc(aL + o, 128 * 16, 128), umma_desc(bH + o, 128 * 16, 128),
                                    1u);
                    }
                    tc2_commit_both(&s_empty[s]);
                }
                __syncwarp();
                continue;
            }
            if (chunk >= X2_NS) mbar_wait(&s_empty[s], (round - 1) & 1u);  // MMAs of chunk - NS done
            uint8_t *sb = stage_base + s * X2_STAGE;
            float2 hx[4], hy[4], hz[4], hzl[4];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int k = k0 + kb * 8 + q;
                const bool ok = k < len;
                const float4 hk = h[ok ? k : 0];
                float zh = hk.z, zl = 0.f;
                if (EXACT_D) two_sum(hk.z, -zref, zh, zl);
                const float xv = ok ? hk.x : 1e30f, yv = ok ? hk.y : 1e30f;
                if (q & 1) {
                    hx[q >> 1].y = xv; hy[q >> 1].y = yv; hz[q >> 1].y = zh; hzl[q >> 1].y = zl;
                } else {
                    hx[q >> 1].x = xv; hy[q >> 1].x = yv; hz[q >> 1].x = zh; hzl[q >> 1].x = zl;
                }
            }
            const float2 nk2 = make_float2(negK, negK);
#pragma unroll
            for (int t = 0; t < X2_NA + X2_NB; ++t) {
                const bool isA = t < X2_NA;
                const float p = isA ? pa[t] : pb[t - X2_NA];
                const float2 mp = make_float2(-p, -p);
                uint32_t wh[4], wl[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const float2 c = isA ? hx[q] : hy[q];
                    const float2 sres =
                        EXACT_D ? __ffma2_rn(mp, hzl[q], __ffma2_rn(mp, hz[q], c)) : __ffma2_rn(mp, hz[q], c);
                    const float2 arg = __fmul2_rn(__fmul2_rn(sres, sres), nk2);
                    const float2 v = make_float2(ex2_approx(arg.x), ex2_approx(arg.y));
                    const float2 vs = __fmul2_rn(v, make_float2(0x1p15f, 0x1p15f));
                    const __half2 hh = __floats2half2_rn(vs.x, vs.y);
                    const float2 hf = __half22float2(hh);                                    // exact
                    const float2 lo = __ffma2_rn(hf, make_float2(-0x1p-15f, -0x1p-15f), v);  // exact
                    const float2 ls = __fmul2_rn(lo, make_float2(0x1p26f, 0x1p26f));
                    wh[q] = *reinterpret_cast<const uint32_t *>(&hh);
                    wl[q] = pack_h2(ls.x, ls.y);
                }
                const int r = lane + 32 * ((isA ? t : t - X2_NA) * X2_NR + rset);
                uint8_t *dh = sb + (isA ? 0 : 2 * X2_PART) + (size_t)(kb * 128 + r) * 16;
                *reinterpret_cast<uint4 *>(dh) = make_uint4(wh[0], wh[1], wh[2], wh[3]);
                *reinterpret_cast<uint4 *>(dh + X2_PART) = make_uint4(wl[0], wl[1], wl[2], wl[3]);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(mapa_rank0(smem_u32(&s_full[s])));
        }
    });

    const int n_chunks = chunk;
    if (mma_warp && rank == 0 && lane == 0) {
        if (n_chunks > 0) tc2_commit_both(&s_done);  // every MMA of the pair tile complete, both CTAs told
    }
    if (n_chunks > 0) mbar_wait(&s_done, 0u);
    tc_fence_after();
    if (!mma_warp) tc_epilogue<MODEL, true>(a, e, t_m, t_n, l, nl, tmem, n_chunks, warp, lane);
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // the peer is done with its TMEM before the pair deallocates
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_N));
}

int tensor16x2_max_stage_hits() { return (227 * 1024 - X2_NS * X2_STAGE - 1024) / 16; }

template <int MODEL, bool ZREF>
static cudaError_t launch_tc16x2(const GridArgs &a0, int n_events, cudaStream_t stream) {
    auto kern = grid_tensor16x2_kernel<MODEL, ZREF>;
    GridArgs a = a0;
    a.cap = min(a.cap, tensor16x2_max_stage_hits()) & ~1;
    const size_t smem = X2_NS * (size_t)X2_STAGE + (size_t)a.cap * sizeof(float4);
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const long long pairs =
        (long long)((a.n0 + 255) / 256) * ((a.n1 + TC_N - 1) / TC_N) * (MODEL == kSlope3 ? a.n2 : 1);
    if (2 * pairs > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        kern<<<dim3((unsigned)(2 * pairs), ne), 32 * (X2_WARPS + 1), smem, stream>>>(a);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

cudaError_t launch_grid_tensor16x2(int model, const GridArgs &a, int n_events, cudaStream_t stream) {
    if (n_events == 0) return cudaSuccess;
    if (model == kSlope3) return launch_tc16x2<kSlope3, false>(a, n_events, stream);
    if (model != kSlope2) return cudaErrorInvalidValue;
    return (a.z_ref == 0.f) ? launch_tc16x2<kSlope2, false>(a, n_events, stream)
                            : launch_tc16x2<kSlope2, true>(a, n_events, stream);
}

int tensor16_max_stage_hits() { return (227 * 1024 - T16_NS * T16_STAGE_BYTES - 1024) / 16; }

template <int MODEL, bool ZREF>
static cudaError_t launch_tc16(const GridArgs &a0, int n_events, cudaStream_t stream) {
    auto kern = grid_tensor16_kernel<MODEL, ZREF>;
    GridArgs a = a0;
    a.cap = min(a.cap, tensor16_max_stage_hits()) & ~1;
    const size_t smem = T16_NS * (size_t)T16_STAGE_BYTES + (size_t)a.cap * sizeof(float4);
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const long long tiles =
        (long long)((a.n0 + TC_M - 1) / TC_M) * ((a.n1 + TC_N - 1) / TC_N) * (MODEL == kSlope3 ? a.n2 : 1);
    if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        kern<<<dim3((unsigned)tiles, ne), 32 * (T16_WARPS + 1), smem, stream>>>(a);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

cudaError_t launch_grid_tensor16(int model, const GridArgs &a, int n_events, cudaStream_t stream) {
    if (n_events == 0) return cudaSuccess;
    if (model == kSlope3) return launch_tc16<kSlope3, false>(a, n_events, stream);
    if (model != kSlope2) return cudaErrorInvalidValue;
    return (a.z_ref == 0.f) ? launch_tc16<kSlope2, false>(a, n_events, stream)
                            : launch_tc16<kSlope2, true>(a, n_events, stream);
}

int tensor_max_stage_hits() {
    // hit slots left after the operand stages, within this CTA's share of the SM
    return (227 * 1024 / RETINA_TC_MINB - 2 * TC_STAGE_BYTES - 1024) / 16;
}

template <int MODEL, bool ZREF>
static cudaError_t launch_tc(const GridArgs &a0, int n_events, cudaStream_t stream) {
    auto kern = grid_tensor_kernel<MODEL, ZREF>;
    GridArgs a = a0;
    a.cap = min(a.cap, tensor_max_stage_hits()) & ~1;
    const size_t smem = 2 * (size_t)TC_STAGE_BYTES + (size_t)a.cap * sizeof(float4);
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const long long tiles =
        (long long)((a.n0 + TC_M - 1) / TC_M) * ((a.n1 + TC_N - 1) / TC_N) * (MODEL == kSlope3 ? a.n2 : 1);
    if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        kern<<<dim3((unsigned)tiles, ne), 32 * TC_WARPS, smem, stream>>>(a);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

cudaError_t launch_grid_tensor(int model, const GridArgs &a, int n_events, cudaStream_t stream) {
    if (n_events == 0) return cudaSuccess;
    if (model == kSlope3) return launch_tc<kSlope3, false>(a, n_events, stream);
    if (model != kSlope2) return cudaErrorInvalidValue;
    return (a.z_ref == 0.f) ? launch_tc<kSlope2, false>(a, n_events, stream)
                            : launch_tc<kSlope2, true>(a, n_events, stream);
}

}  // namespace retina
