// grid_tensor16p.cu -- EXPERIMENTAL persistent variant of the fp16-split grid kernel
// (-DRETINA_T16_PERSISTENT=1; default off).  Eq. (2) as a dense contraction over hits on the
// tcgen05 tensor cores with fp16 operands (kind::f16), persistent and warp-specialised.
// Measured (parity green on every tensor test) but SLOWER than the one-CTA-per-tile kernel
// grid_tensor16_kernel: cfg3 10.6 vs 7.4 ms, cfg4 38 vs 15.4 ms per 1000 / 50 events -- the
// third fp16 part adds generation work where generation, not the tensor pipe, is the limit, and
// SLOPE3's z0-fastest 4-byte stores no longer meet in L2 across concurrently running CTAs.
//
//     R[i][j] = sum_k EX[i][k] EY[j][k],  EX = 2^(-K (x - tx z)^2),  EY = 2^(-K (y - ty z)^2)
//
// (the exact factorisation of exp(-s^2/sigma^2) for the in-plane distance).
//
// Exact fp16 split with ONE accumulator.  Every factor v in [0, 1] is written as
//     v = h + l,   h = fp16_rn(v 2^15) 2^-15 (exact back in fp32),   l = v - h (exact, |l| <= 2^-12 v),
// and each operand row carries three fp16 parts, scaled so that all three products land on the
// same scale 2^30 and accumulate into one fp32 TMEM accumulator:
//     A = [h 2^15 | h 2^9  | l 2^21],   B = [h 2^15 | l 2^21 | h 2^9]
//     A.B = 2^30 (h_x h_y + h_x l_y + l_x h_y)            R = D 2^-30.
// Dropped: l_x l_y (<= 2^-24 relative).  fp16 rounding of l 2^21: <= 2^-24 relative of v, and where
// a part falls below the fp16 normal range the absolute error stays <= 2^-45 per term (h 2^9 is
// normal for h >= 2^-23, l 2^21 for l >= 2^-35) -- far below the T1 floor (1e-11 per cell).
//
// Persistent CTA per SM over a contiguous range of (event, tile[, z0]) work items (z0 fastest, so
// one CTA writes neighbouring z0 values of the same cells back to back):
//   warps 0-15  generate: per 32-hit chunk, warp w writes the 8-hit k-block w % 4 (16 B per row
//               and part) of 1 A row and 2 B rows per lane into stage c % NS, then arrives on
//               full[stage]; hits are read straight from global memory (L1-resident per event);
//   warp  16    issues the 6 MMAs (M=128, N=256, K=16) of each chunk into the tile's accumulator
//               buffer and commits them to empty[stage]; at the end of a tile it commits acc_full;
//   warps 17-20 epilogue: TMEM -> registers (tcgen05.ld 32x32b.x16) -> global, then acc_empty.
// TMEM: two 128 x 256 fp32 accumulators (all 512 columns), so the epilogue of tile i overlaps the
// MMAs of tile i+1.
#include "common.cuh"
#include "kernels.cuh"
#include "tcgen05.cuh"

#include <cuda_fp16.h>

#include <algorithm>

namespace retina {

#ifndef RETINA_P16_NS
#define RETINA_P16_NS 2
#endif
constexpr int P16_KC = 32;                           // hits per chunk
constexpr int P16_NS = RETINA_P16_NS;                // operand stages in the ring
constexpr int P16_KB = P16_KC / 8;                   // 8-hit k-blocks per chunk
constexpr int P16_PART_A = TC_M * P16_KC * 2;        // one fp16 part of A: 8 KB
constexpr int P16_PART_B = TC_N * P16_KC * 2;        // one fp16 part of B: 16 KB
constexpr int P16_STAGE = 3 * P16_PART_A + 3 * P16_PART_B;  // 72 KB
constexpr int P16_GEN_WARPS = 16;
constexpr int P16_MMA_WARP = P16_GEN_WARPS;
constexpr int P16_WARPS = P16_GEN_WARPS + 1 + 4;
constexpr int P16_NR = P16_GEN_WARPS / P16_KB;       // row sets per k-block (4)
constexpr int P16_NA = 4 / P16_NR, P16_NB = 8 / P16_NR;  // A and B rows per lane per chunk (1, 2)
static_assert(P16_NS * P16_STAGE + 1024 <= 227 * 1024, "operand ring exceeds shared memory");

__device__ __forceinline__ void mbar_arrive1(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct TileCoord {
    int e, l, t_m, t_n;
};

__device__ __forceinline__ TileCoord decode_tile(int t, int tpe, int nl, int tn) {
    TileCoord c;
    c.e = t / tpe;
    const int r = t - c.e * tpe;
    c.l = r % nl;
    const int tile = r / nl;
    c.t_n = tile % tn;
    c.t_m = tile / tn;
    return c;
}

template <int MODEL, bool ZREF>
__global__ void __launch_bounds__(32 * P16_WARPS, 1) grid_tensor16p_kernel(GridArgs a, int n_items) {
    extern __shared__ __align__(1024) uint8_t s_raw[];
    __shared__ __align__(8) uint64_t s_full[P16_NS];
    __shared__ __align__(8) uint64_t s_empty[P16_NS];
    __shared__ __align__(8) uint64_t s_acc_full[2];
    __shared__ __align__(8) uint64_t s_acc_empty[2];
    __shared__ uint32_t s_tmem;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tn = (a.n1 + TC_N - 1) / TC_N, tm = (a.n0 + TC_M - 1) / TC_M;
    const int nl = (MODEL == kSlope3) ? a.n2 : 1;
    const int tpe = tm * tn * nl;  // work items per event
    const int t0 = (int)((long long)blockIdx.x * n_items / gridDim.x);
    const int t1 = (int)((long long)(blockIdx.x + 1) * n_items / gridDim.x);

    if (warp == 0) {  // two accumulator buffers: 128 lanes x (256 + 256) fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(2 * TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        tc_fence_before();
    }
    if (tid == 0) {
        for (int i = 0; i < P16_NS; ++i) {
            mbar_init(&s_full[i], P16_GEN_WARPS);
            mbar_init(&s_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_acc_full[i], 1);
            mbar_init(&s_acc_empty[i], 4);
        }
        fence_mbar_init();
    }
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t stage_saddr = smem_u32(s_raw);
    constexpr bool EXACT_D = ZREF || MODEL == kSlope3;

    if (warp < P16_GEN_WARPS) {
        // ------------------------------------------------------------------ generating warps
        const int kb = warp % P16_KB, rset = warp / P16_KB;
        const float2 nk2 = make_float2(a.negK, a.negK);
        const __half2 h2m6 = __float2half2_rn(0.015625f);  // 2^-6: h 2^15 -> h 2^9 (exact in range)
        uint32_t cg = 0;                                   // chunk counter (ring position)
        for (int t = t0; t < t1; ++t) {
            const TileCoord c = decode_tile(t, tpe, nl, tn);
            const int start = a.offsets[c.e], n = a.offsets[c.e + 1] - start;
            if (n <= 0) continue;
            const float4 *hg = a.hits + start;
            float p[P16_NA + P16_NB];
#pragma unroll
            for (int u = 0; u < P16_NA; ++u)
                p[u] = __ldg(a.nodes0 + min(c.t_m * TC_M + lane + 32 * (u * P16_NR + rset), a.n0 - 1));
#pragma unroll
            for (int u = 0; u < P16_NB; ++u)
                p[P16_NA + u] = __ldg(a.nodes1 + min(c.t_n * TC_N + lane + 32 * (u * P16_NR + rset), a.n1 - 1));
            const float zref = (MODEL == kSlope3) ? __ldg(a.nodes2 + c.l) : a.z_ref;
            for (int k0 = 0; k0 < n; k0 += P16_KC, ++cg) {
                const int s = (int)(cg % P16_NS);
                // hits of this warp's k-block as pairs (q, q+1); a missing hit gets a huge
                // coordinate so its factor is exactly ex2(-inf) = 0
                float2 hx[4], hy[4], hz[4], hzl[4];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int k = k0 + kb * 8 + q;
                    const bool ok = k < n;
                    const float4 hk = __ldg(hg + (ok ? k : 0));
                    float zh = hk.z, zl = 0.f;
                    if (EXACT_D) two_sum(hk.z, -zref, zh, zl);
                    const float xv = ok ? hk.x : 1e30f, yv = ok ? hk.y : 1e30f;
                    if (q & 1) {
                        hx[q >> 1].y = xv; hy[q >> 1].y = yv; hz[q >> 1].y = zh; hzl[q >> 1].y = zl;
                    } else {
                        hx[q >> 1].x = xv; hy[q >> 1].x = yv; hz[q >> 1].x = zh; hzl[q >> 1].x = zl;
                    }
                }
                if (cg >= P16_NS) mbar_wait(&s_empty[s], ((cg / P16_NS) - 1) & 1u);  // MMAs of cg-NS done
                uint8_t *sb = s_raw + s * P16_STAGE;
#pragma unroll
                for (int u = 0; u < P16_NA + P16_NB; ++u) {
                    const bool isA = u < P16_NA;
                    const float2 mp = make_float2(-p[u], -p[u]);
                    uint32_t w15[4], wlo[4], w9[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float2 cc = isA ? hx[q] : hy[q];
                        const float2 sres =
                            EXACT_D ? __ffma2_rn(mp, hzl[q], __ffma2_rn(mp, hz[q], cc)) : __ffma2_rn(mp, hz[q], cc);
                        const float2 arg = __fmul2_rn(__fmul2_rn(sres, sres), nk2);
                        const float2 v = make_float2(ex2_approx(arg.x), ex2_approx(arg.y));
                        const float2 vs = __fmul2_rn(v, make_float2(0x1p15f, 0x1p15f));
                        const __half2 hh = __floats2half2_rn(vs.x, vs.y);
                        const float2 hf = __half22float2(hh);                                    // exact
                        const float2 lo = __ffma2_rn(hf, make_float2(-0x1p-15f, -0x1p-15f), v);  // exact
                        const float2 ls = __fmul2_rn(lo, make_float2(0x1p21f, 0x1p21f));
                        const __half2 hl = __floats2half2_rn(ls.x, ls.y);
                        const __half2 h9 = __hmul2(hh, h2m6);
                        w15[q] = *reinterpret_cast<const uint32_t *>(&hh);
                        wlo[q] = *reinterpret_cast<const uint32_t *>(&hl);
                        w9[q] = *reinterpret_cast<const uint32_t *>(&h9);
                    }
                    // K-major no-swizzle canonical layout: k-block kb of 8 fp16, row r at 16 B
                    const int r = lane + 32 * ((isA ? u : u - P16_NA) * P16_NR + rset);
                    const int rows = isA ? TC_M : TC_N;
                    const int part = isA ? P16_PART_A : P16_PART_B;
                    uint8_t *d0 = sb + (isA ? 0 : 3 * P16_PART_A) + (size_t)(kb * rows + r) * 16;
                    // A = [h 2^15 | h 2^9 | l 2^21],  B = [h 2^15 | l 2^21 | h 2^9]
                    *reinterpret_cast<uint4 *>(d0) = make_uint4(w15[0], w15[1], w15[2], w15[3]);
                    *reinterpret_cast<uint4 *>(d0 + part) =
                        isA ? make_uint4(w9[0], w9[1], w9[2], w9[3]) : make_uint4(wlo[0], wlo[1], wlo[2], wlo[3]);
                    *reinterpret_cast<uint4 *>(d0 + 2 * part) =
                        isA ? make_uint4(wlo[0], wlo[1], wlo[2], wlo[3]) : make_uint4(w9[0], w9[1], w9[2], w9[3]);
                }
                fence_proxy_async();  // this thread's generic-proxy stores -> visible to the tensor core
                __syncwarp();
                if (lane == 0) mbar_arrive1(&s_full[s]);
            }
        }
    } else if (warp == P16_MMA_WARP) {
        // ------------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            uint32_t cg = 0;
            int ti = 0;
            for (int t = t0; t < t1; ++t, ++ti) {
                const TileCoord c = decode_tile(t, tpe, nl, tn);
                const int n = a.offsets[c.e + 1] - a.offsets[c.e];
                const int b = ti & 1;
                if (ti >= 2) mbar_wait(&s_acc_empty[b], ((ti >> 1) - 1) & 1);  // epilogue of tile ti-2 done
                tc_fence_after();
                const uint32_t acc = tmem + (uint32_t)(b * TC_N);
                const int nck = n > 0 ? (n + P16_KC - 1) / P16_KC : 0;
                for (int ck = 0; ck < nck; ++ck, ++cg) {
                    const int s = (int)(cg % P16_NS);
                    mbar_wait(&s_full[s], (cg / P16_NS) & 1u);
                    tc_fence_after();
                    const uint32_t A0 = stage_saddr + s * P16_STAGE, B0 = A0 + 3 * P16_PART_A;
#pragma unroll
                    for (int j = 0; j < P16_KC / 16; ++j) {  // K = 16 fp16 per MMA = 2 k-blocks
                        const uint32_t oa = j * 2 * (TC_M * 16), ob = j * 2 * (TC_N * 16);
#pragma unroll
                        for (int pp = 0; pp < 3; ++pp)
                            tc_mma_f16(acc, umma_desc(A0 + pp * P16_PART_A + oa, TC_M * 16, 128),
                                       umma_desc(B0 + pp * P16_PART_B + ob, TC_N * 16, 128),
                                       (ck > 0 || j > 0 || pp > 0) ? 1u : 0u);
                    }
                    tc_commit(&s_empty[s]);
                }
                if (nck > 0)
                    tc_commit(&s_acc_full[b]);  // arrives when every MMA of this tile is complete
                else
                    mbar_arrive1(&s_acc_full[b]);
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------------ epilogue warps
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        int ti = 0;
        for (int t = t0; t < t1; ++t, ++ti) {
            const TileCoord c = decode_tile(t, tpe, nl, tn);
            const int n = a.offsets[c.e + 1] - a.offsets[c.e];
            const int b = ti & 1;
            mbar_wait(&s_acc_full[b], (ti >> 1) & 1);
            tc_fence_after();
            const int i = c.t_m * TC_M + q * 32 + lane;
            const int64_t cells = (int64_t)a.n0 * a.n1 * nl;
            float *out = a.R + (int64_t)(a.e_base + c.e) * cells + (int64_t)i * a.n1 * nl;
#pragma unroll 1
            for (int cc = 0; cc < TC_N / 16; ++cc) {
                const int col = cc * 16;
                uint32_t v[16];
                if (n > 0) {
                    const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * TC_N + col);
                    asm volatile(
                        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
                        "%15}, [%16];"
                        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
                          "=r"(v[14]), "=r"(v[15])
                        : "r"(taddr));
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int x = 0; x < 16; ++x) v[x] = __float_as_uint(__fmul_rn(__uint_as_float(v[x]), 0x1p-30f));
                } else {
#pragma unroll
                    for (int x = 0; x < 16; ++x) v[x] = 0u;
                }
                const int j0 = c.t_n * TC_N + col;
                if (i < a.n0 && MODEL == kSlope3) {
#pragma unroll
                    for (int x = 0; x < 16; ++x)
                        if (j0 + x < a.n1) out[(int64_t)(j0 + x) * nl + c.l] = __uint_as_float(v[x]);
                } else if (i < a.n0) {
                    if (j0 + 15 < a.n1 && (((uintptr_t)(out + j0)) & 15u) == 0) {
#pragma unroll
                        for (int x = 0; x < 16; x += 4)
                            *reinterpret_cast<float4 *>(out + j0 + x) =
                                make_float4(__uint_as_float(v[x]), __uint_as_float(v[x + 1]),
                                            __uint_as_float(v[x + 2]), __uint_as_float(v[x + 3]));
                    } else {
#pragma unroll
                        for (int x = 0; x < 16; ++x)
                            if (j0 + x < a.n1) out[j0 + x] = __uint_as_float(v[x]);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive1(&s_acc_empty[b]);
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_N));
    }
}

static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0, v = 0;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) ==
                                                       cudaSuccess)
            n = v;
        if (n <= 0) n = 148;
    }
    return n;
}

template <int MODEL, bool ZREF>
static cudaError_t launch_p16(const GridArgs &a0, int n_events, cudaStream_t stream) {
    auto kern = grid_tensor16p_kernel<MODEL, ZREF>;
    const size_t smem = (size_t)P16_NS * P16_STAGE;
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const long long per_event =
        (long long)((a0.n0 + TC_M - 1) / TC_M) * ((a0.n1 + TC_N - 1) / TC_N) * (MODEL == kSlope3 ? a0.n2 : 1);
    // work items are int32: split the batch into launches of at most 2^31-1 items
    const int ev_per_launch = (int)std::max(1LL, std::min((long long)n_events, 0x7fffffffLL / per_event));
    for (int e0 = 0; e0 < n_events; e0 += ev_per_launch) {
        GridArgs a = a0;
        const int ne = std::min(ev_per_launch, n_events - e0);
        a.offsets = a0.offsets + e0;  // event e of this launch = e0 + e of the batch
        a.e_base = e0;
        const int items = (int)(per_event * ne);
        const int grid = std::min(items, sm_count());
        kern<<<grid, 32 * P16_WARPS, smem, stream>>>(a, items);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

cudaError_t launch_grid_tensor16p(int model, const GridArgs &a, int n_events, cudaStream_t stream) {
    if (n_events == 0) return cudaSuccess;
    if (model == kSlope3) return launch_p16<kSlope3, false>(a, n_events, stream);
    if (model != kSlope2) return cudaErrorInvalidValue;
    return (a.z_ref == 0.f) ? launch_p16<kSlope2, false>(a, n_events, stream)
                            : launch_p16<kSlope2, true>(a, n_events, stream);
}

}  // namespace retina
