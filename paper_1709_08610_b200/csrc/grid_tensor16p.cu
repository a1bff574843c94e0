// grid_tensor16p.cu -- K1h, the default grid kernel for SLOPE2 / SLOPE3 (RETINA_GRID_TENSOR_F16,
// what RETINA_GRID_AUTO runs): persistent CTA-pair variant of the fp16-split grid kernel.  Eq. (2)
// as a dense contraction over hits on the tcgen05 tensor cores (kind::f16, cta_group::2, M = 256),
// with the per-tile prologue and epilogue taken off the MMA critical path:
//
//     R[i][j] = sum_k EX[i][k] EY[j][k],  EX = 2^(-K (x - tx z)^2),  EY = 2^(-K (y - ty z)^2)
//
// (the exact factorisation of exp(-s^2/sigma^2) for the in-plane distance).
//
// Exact fp16 split with ONE accumulator, so that two accumulators fit TMEM and the epilogue of
// tile i overlaps the MMAs of tile i+1.  Every factor v in [0, 1] is written as
//     v = h + l,   h = fp16_rn(v 2^15) 2^-15 (exact back in fp32),   l = v - h (exact, |l| <= 2^-12 v),
// and each operand row carries three fp16 parts, scaled so that the three products share the
// scale 2^30 and accumulate into one fp32 TMEM accumulator:
//     A = [h 2^15 | h 2^9  | l 2^21],   B = [h 2^15 | l 2^21 | h 2^9]
//     A.B = 2^30 (h_x h_y + h_x l_y + l_x h_y)            R = D 2^-30.
// Dropped: l_x l_y (<= 2^-24 relative).  fp16 rounding of l 2^21: <= 2^-24 relative of v; where a
// part falls below the fp16 normal range (h 2^9 for h < 2^-23, l 2^21 for l < 2^-35) the absolute
// error stays <= 2^-45 per term -- far below the T1 floor (1e-11 per cell).
//
// A cluster of two CTAs (one TPC) loops over a contiguous range of (event, [z0 plane,] 256 x 256
// pair tile) work items, so an event's hits are loaded once per cluster.  Every item writes whole
// row segments (1 KB per row) of one [n0][n1] plane: a SLOPE3 grid is stored z0 plane by z0 plane
// (Z37).  Per CTA (rank r):
//   warps 0-15  generate its 128 A rows (tx) and its half of B (128 ty rows) per 64-hit chunk
//               into stage c % NS, then arrive on the even CTA's full[stage] (cluster arrive);
//               hits live in shared memory, reloaded only when the event changes (or windowed
//               when an event exceeds the stage);
//   warp  16    (even CTA) issues the chunk's 6 MMAs (M = 256, N = 256, K = 16) into the tile's
//               accumulator buffer, commits empty[stage] to both CTAs, and acc_full at tile end;
//   warps 17-20 epilogue of its 128 rows: TMEM -> registers -> global, then a cluster arrive on
//               the even CTA's acc_empty[buffer].
#include "common.cuh"
#include "kernels.cuh"
#include "tcgen05.cuh"

#include <cuda.h>           // CUtensorMap (the encoder is fetched from the driver at run time)
#include <cudaTypedefs.h>   // PFN_cuTensorMapEncodeTiled

#include <algorithm>

namespace retina {

#ifndef RETINA_PP_KC
#define RETINA_PP_KC 64
#endif
#ifndef RETINA_PP_NS
#define RETINA_PP_NS 2
#endif
constexpr int PP_KC = RETINA_PP_KC;                 // hits per chunk
constexpr int PP_NS = RETINA_PP_NS;                 // operand stages in the ring
constexpr int PP_KB = PP_KC / 8;                    // 8-hit k-blocks per chunk
constexpr int PP_PART = 128 * PP_KC * 2;            // one fp16 part of A or of this CTA's B half
constexpr int PP_STAGE = 6 * PP_PART;               // A: 3 parts, B half: 3 parts
constexpr int PP_GEN_WARPS = 16;
constexpr int PP_MMA_WARP = PP_GEN_WARPS;
constexpr int PP_WARPS = PP_GEN_WARPS + 1 + 4;
constexpr int PP_NR = PP_GEN_WARPS / PP_KB;         // row sets per k-block
constexpr int PP_NA = 4 / PP_NR, PP_NB = 4 / PP_NR; // A and B rows per lane per chunk
static_assert(PP_NR >= 1 && 4 % PP_NR == 0, "warps / k-blocks must divide the 4 row groups");
static_assert(PP_KC % 16 == 0, "K = 16 per kind::f16 MMA");
static_assert(PP_NS * PP_STAGE + 2048 + 64 * 16 <= 227 * 1024, "operand ring must leave room for hits");

struct PairCoord {
    int e, l, t_m, t_n;  // event (of this launch), z0 index, 128-row block of tx, 256-column block of ty
};

__device__ __forceinline__ PairCoord decode_pair(int t, int ppe, int nl, int tn, int rank) {
    PairCoord c;
    c.e = t / ppe;
    const int r = t - c.e * ppe;
    c.l = r % nl;
    const int tile = r / nl;
    c.t_n = tile % tn;
    c.t_m = 2 * (tile / tn) + rank;
    return c;
}

__device__ __forceinline__ void gen_bar_sync() {  // the 16 generating warps only
    asm volatile("bar.sync 1, %0;" ::"n"(32 * PP_GEN_WARPS) : "memory");
}

// Epilogue staging for the TMA tensor store: per epilogue warp two 32-row x 16-column fp32 boxes
// (2 KB each, 64-byte swizzle: 16-byte chunk c of row r at r 64 + ((c ^ ((r >> 1) & 3)) << 4), so the
// warp's row-per-lane STS.128s are bank-conflict-free).
constexpr int PP_EPI_BOX = 32 * 16 * 4;
constexpr int PP_EPI_BYTES = 4 * 2 * PP_EPI_BOX;

// least |x - t d| over t in [t0, t1] and d in [d0, d1] (0 when the range of t d contains x); the
// products' range is widened by 1e-6 of its magnitude so it holds every exact t d
__device__ __forceinline__ float pp_min_abs(float x, float t0, float t1, float d0, float d1) {
    const float p00 = t0 * d0, p01 = t0 * d1, p10 = t1 * d0, p11 = t1 * d1;
    const float pmin = fminf(fminf(p00, p01), fminf(p10, p11)), pmax = fmaxf(fmaxf(p00, p01), fmaxf(p10, p11));
    const float slack = 1e-6f * fmaxf(fabsf(pmin), fabsf(pmax));
    const float lo = x - (pmax + slack), hi = x - (pmin - slack);
    return (lo > 0.f) ? lo : (hi < 0.f ? -hi : 0.f);
}

// CULL (RETINA_GRID_TENSOR_F16_CULLED): per pair tile, the hit window holds only the hits that can
// reach the tile -- a conservative bound puts K s^2 <= 128 for some (tx, ty) of the tile, i.e. a
// product e_x e_y >= 2^-128 -- in hit order; every other hit's contribution to every cell of the
// tile is below 2^-128 (fp32's normal range ends at 2^-126).  Windows are then per tile, and each
// chunk carries a "last of its tile" flag for the MMA warp and the relay.
template <int MODEL, bool ZREF, bool TMA_EPI, bool CULL = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * PP_WARPS)
    grid_tensor16pp_kernel(GridArgs a, int n_items, const __grid_constant__ CUtensorMap out_map) {
    extern __shared__ __align__(1024) uint8_t s_raw[];
    __shared__ __align__(8) uint64_t s_full[PP_NS];     // even CTA: its 16 generating warps + the odd CTA's relay
    __shared__ __align__(8) uint64_t s_pfull[PP_NS];    // odd CTA: its 16 generating warps (relayed once)
    __shared__ __align__(8) uint64_t s_empty[PP_NS];    // both CTAs: multicast MMA commit
    __shared__ __align__(8) uint64_t s_acc_full[2];     // both CTAs: multicast commit at tile end
    __shared__ __align__(8) uint64_t s_acc_empty[2];    // even CTA: 2 x 4 epilogue warps arrive
    __shared__ uint32_t s_tmem;
    __shared__ int s_last[PP_NS];                        // CULL: stage holds its tile's last chunk
    __shared__ int s_wcnt[PP_GEN_WARPS];                 // CULL: kept hits per generating warp, per round

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rank = cluster_rank();
    const int tn = (a.n1 + TC_N - 1) / TC_N, pm = (a.n0 + 255) / 256;
    const int nl = (MODEL == kSlope3) ? a.n2 : 1;
    const int ppe = pm * tn * nl;  // pair work items per event
    const int cl = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    // a contiguous range of items per cluster (the event's hits stay in shared memory)
    const int t0 = (int)((long long)cl * n_items / ncl), t1 = (int)((long long)(cl + 1) * n_items / ncl);
    constexpr int dt = 1;
    constexpr bool EXACT_D = ZREF || MODEL == kSlope3;
    // [operand stages][epilogue boxes (TMA_EPI)][hit window]; the hit window is a structure of
    // arrays: x, y, z - z_ref (hi) [, lo], a.cap floats each
    uint8_t *s_epi = s_raw + PP_NS * PP_STAGE;
    float *s_hx = reinterpret_cast<float *>(s_epi + (TMA_EPI ? PP_EPI_BYTES : 0));
    float *s_hy = s_hx + a.cap, *s_hz = s_hy + a.cap, *s_hzl = s_hz + a.cap;

    if (warp == 0) {  // two accumulator buffers of 128 lanes x 256 fp32 columns, in both CTAs
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(2 * TC_N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        tc_fence_before();
    }
    if (tid == 0) {
        for (int i = 0; i < PP_NS; ++i) {
            mbar_init(&s_full[i], PP_GEN_WARPS + 1);
            mbar_init(&s_pfull[i], PP_GEN_WARPS);
            mbar_init(&s_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_acc_full[i], 1);
            mbar_init(&s_acc_empty[i], 8);
        }
        fence_mbar_init();
    }
    __syncthreads();
    cluster_sync_all();  // the peer's barriers exist before any remote arrive
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    const uint32_t stage_saddr = smem_u32(s_raw);

    if (warp < PP_GEN_WARPS) {
        // ------------------------------------------------------------------ generating warps
        const int kb = warp % PP_KB, rset = warp / PP_KB;
        const int gtid = tid;  // 0 .. 32 * PP_GEN_WARPS - 1
        // 2^15 is folded into the exponent: v' = 2^(15 - K s^2) = v 2^15 straight from MUFU.EX2
        const float2 nk2 = make_float2(a.negK, a.negK), c15 = make_float2(15.f, 15.f);
        const __half2 h2m6 = __float2half2_rn(0.015625f);  // 2^-6: h 2^15 -> h 2^9
        uint32_t cg = 0;                                   // chunk counter
        int have_e = -1, have_w0 = -1, have_l = -1;        // hit window (and z0) now in shared memory
        // each warp arrives on a barrier of its own CTA (CTA-scope release: cheap); the odd CTA's
        // arrivals are relayed to the even CTA by one cluster-scope release per chunk (MMA warp)
        uint64_t *arrive_bar = (rank == 0) ? s_full : s_pfull;
        for (int t = t0; t < t1; t += dt) {
            const PairCoord c = decode_pair(t, ppe, nl, tn, (int)rank);
            const int start = a.offsets[c.e], n = a.offsets[c.e + 1] - start;
            float p[PP_NA + PP_NB];
#pragma unroll
            for (int u = 0; u < PP_NA; ++u)
                p[u] = __ldg(a.nodes0 + min(c.t_m * 128 + lane + 32 * (u * PP_NR + rset), a.n0 - 1));
#pragma unroll
            for (int u = 0; u < PP_NB; ++u)  // this CTA's half of the pair tile's 256 ty columns
                p[PP_NA + u] =
                    __ldg(a.nodes1 + min(c.t_n * TC_N + (int)rank * 128 + lane + 32 * (u * PP_NR + rset), a.n1 - 1));
            const float zref = (MODEL == kSlope3) ? __ldg(a.nodes2 + c.l) : a.z_ref;
            // CULL: the pair tile's parameter box (both CTAs: the same box, so the same lists)
            float txl = 0.f, txh = 0.f, tyl = 0.f, tyh = 0.f;
            if (CULL) {
                const int i0 = (c.t_m & ~1) * 128, j0 = c.t_n * TC_N;
                const float u0 = __ldg(a.nodes0 + i0), u1 = __ldg(a.nodes0 + min(i0 + 255, a.n0 - 1));
                const float v0 = __ldg(a.nodes1 + j0), v1 = __ldg(a.nodes1 + min(j0 + TC_N - 1, a.n1 - 1));
                txl = fminf(u0, u1);
                txh = fmaxf(u0, u1);
                tyl = fminf(v0, v1);
                tyh = fmaxf(v0, v1);
            }
            const float K = -a.negK;
            int r0 = 0;             // CULL: next raw hit of the event to scan
            long long kept = 0;     // CULL: hits this tile keeps (all windows)
            for (int w0 = 0; CULL ? (r0 < n) : (w0 < n); w0 += a.cap) {
                int wlen = min(a.cap, n - w0);
                if (CULL) {
                    // scan rounds of 512 raw hits, keeping (in hit order) those within reach of the
                    // tile, until the window would overflow or the event is done
                    int L = 0;
                    while (r0 < n) {
                        const int k = r0 + gtid;
                        float4 hk = make_float4(0.f, 0.f, 0.f, 0.f);
                        bool keep = false;
                        if (k < n) {
                            hk = __ldg(a.hits + start + k);
                            const float d0 = (EXACT_D) ? __fsub_rd(hk.z, zref) : hk.z;
                            const float d1 = (EXACT_D) ? __fsub_ru(hk.z, zref) : hk.z;
                            const float mx = pp_min_abs(hk.x, txl, txh, d0, d1);
                            const float my = pp_min_abs(hk.y, tyl, tyh, d0, d1);
                            keep = K * __fmaf_rn(mx, mx, my * my) * 0.99999f <= 128.f;
                        }
                        const unsigned bal = __ballot_sync(0xffffffffu, keep);
                        gen_bar_sync();  // the previous round's counts are read
                        if (lane == 0) s_wcnt[warp] = __popc(bal);
                        gen_bar_sync();
                        int off = 0, tot = 0;
#pragma unroll
                        for (int w = 0; w < PP_GEN_WARPS; ++w) {
                            const int cw = s_wcnt[w];
                            off += (w < warp) ? cw : 0;
                            tot += cw;
                        }
                        if (L + tot > a.cap) break;  // the round goes to the next window
                        if (keep) {
                            const int o = L + off + __popc(bal & ((1u << lane) - 1u));
                            float zh = hk.z, zl = 0.f;
                            if (EXACT_D) two_sum(hk.z, -zref, zh, zl);
                            s_hx[o] = hk.x;
                            s_hy[o] = hk.y;
                            s_hz[o] = zh;
                            if (EXACT_D) s_hzl[o] = zl;
                        }
                        L += tot;
                        r0 += 32 * PP_GEN_WARPS;
                    }
                    // pad to whole chunks (at least one: an item whose window is empty still runs one
                    // chunk of far-away hits, so the MMA warp writes its accumulator with zeros)
                    const int Lpad = max(PP_KC, (L + PP_KC - 1) / PP_KC * PP_KC);
                    for (int k = L + gtid; k < Lpad; k += 32 * PP_GEN_WARPS) {
                        s_hx[k] = 1e30f;
                        s_hy[k] = 1e30f;
                        s_hz[k] = 0.f;
                        if (EXACT_D) s_hzl[k] = 0.f;
                    }
                    gen_bar_sync();
                    wlen = max(L, 1);
                    kept += L;
                    have_e = -1;  // the dense path's window is gone
                } else if (have_e != c.e || have_w0 != w0 || (MODEL == kSlope3 && have_l != c.l)) {
                    // (re)stage the window as structure-of-arrays x, y, z - z_ref (exact as zh + zl),
                    // padded to whole chunks with far-away hits (x = y = 1e30: factor 0), so each
                    // thread loads its 8 hits' coordinates as aligned float4s straight into the
                    // register pairs the FFMA2s use; uniform over the 16 warps
                    gen_bar_sync();  // nobody still reads the old window
                    const int wpad = (wlen + PP_KC - 1) / PP_KC * PP_KC;
                    RETINA_ASSERT(wpad <= a.cap);
                    for (int k = gtid; k < wpad; k += 32 * PP_GEN_WARPS) {
                        float x = 1e30f, y = 1e30f, zh = 0.f, zl = 0.f;
                        if (k < wlen) {
                            const float4 hk = __ldg(a.hits + start + w0 + k);
                            x = hk.x;
                            y = hk.y;
                            zh = hk.z;
                            if (EXACT_D) two_sum(hk.z, -zref, zh, zl);
                        }
                        s_hx[k] = x;
                        s_hy[k] = y;
                        s_hz[k] = zh;
                        if (EXACT_D) s_hzl[k] = zl;
                    }
                    gen_bar_sync();
                    have_e = c.e;
                    have_w0 = w0;
                    have_l = c.l;
                }
                for (int k0 = 0; k0 < wlen; k0 += PP_KC, ++cg) {
                    const int s = (int)(cg % PP_NS);
                    const int kk = k0 + kb * 8;
                    RETINA_ASSERT(kk + 8 <= a.cap);
                    float2 hx[4], hy[4], hz[4], hzl[4];
                    {
                        const float4 x0 = *reinterpret_cast<const float4 *>(s_hx + kk);
                        const float4 x1 = *reinterpret_cast<const float4 *>(s_hx + kk + 4);
                        const float4 y0 = *reinterpret_cast<const float4 *>(s_hy + kk);
                        const float4 y1 = *reinterpret_cast<const float4 *>(s_hy + kk + 4);
                        const float4 z0 = *reinterpret_cast<const float4 *>(s_hz + kk);
                        const float4 z1 = *reinterpret_cast<const float4 *>(s_hz + kk + 4);
                        hx[0] = make_float2(x0.x, x0.y); hx[1] = make_float2(x0.z, x0.w);
                        hx[2] = make_float2(x1.x, x1.y); hx[3] = make_float2(x1.z, x1.w);
                        hy[0] = make_float2(y0.x, y0.y); hy[1] = make_float2(y0.z, y0.w);
                        hy[2] = make_float2(y1.x, y1.y); hy[3] = make_float2(y1.z, y1.w);
                        hz[0] = make_float2(z0.x, z0.y); hz[1] = make_float2(z0.z, z0.w);
                        hz[2] = make_float2(z1.x, z1.y); hz[3] = make_float2(z1.z, z1.w);
                        if (EXACT_D) {
                            const float4 l0 = *reinterpret_cast<const float4 *>(s_hzl + kk);
                            const float4 l1 = *reinterpret_cast<const float4 *>(s_hzl + kk + 4);
                            hzl[0] = make_float2(l0.x, l0.y); hzl[1] = make_float2(l0.z, l0.w);
                            hzl[2] = make_float2(l1.x, l1.y); hzl[3] = make_float2(l1.z, l1.w);
                        }
                    }
                    if (cg >= PP_NS) mbar_wait(&s_empty[s], ((cg / PP_NS) - 1) & 1u);  // MMAs of cg-NS done
                    uint8_t *sb = s_raw + s * PP_STAGE;
#pragma unroll
                    for (int u = 0; u < PP_NA + PP_NB; ++u) {
                        const bool isA = u < PP_NA;
                        const float2 mp = make_float2(-p[u], -p[u]);
                        uint32_t w15[4], wlo[4], w9[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const float2 cc = isA ? hx[q] : hy[q];
                            const float2 sres = EXACT_D ? __ffma2_rn(mp, hzl[q], __ffma2_rn(mp, hz[q], cc))
                                                        : __ffma2_rn(mp, hz[q], cc);
                            const float2 arg = __ffma2_rn(__fmul2_rn(sres, sres), nk2, c15);
                            const float2 vs = make_float2(ex2_approx(arg.x), ex2_approx(arg.y));  // v 2^15
                            const __half2 hh = __floats2half2_rn(vs.x, vs.y);
                            const float2 hf = __half22float2(hh);                                  // exact
                            const float2 lo = __ffma2_rn(hf, make_float2(-1.f, -1.f), vs);         // exact
                            const float2 ls = __fmul2_rn(lo, make_float2(0x1p6f, 0x1p6f));       // l 2^21
                            const __half2 hl = __floats2half2_rn(ls.x, ls.y);
                            const __half2 h9 = __hmul2(hh, h2m6);
                            w15[q] = *reinterpret_cast<const uint32_t *>(&hh);
                            wlo[q] = *reinterpret_cast<const uint32_t *>(&hl);
                            w9[q] = *reinterpret_cast<const uint32_t *>(&h9);
                        }
                        // K-major no-swizzle canonical layout: k-block kb of 8 fp16, row r at 16 B
                        const int r = lane + 32 * ((isA ? u : u - PP_NA) * PP_NR + rset);
                        uint8_t *d0 = sb + (isA ? 0 : 3 * PP_PART) + (size_t)(kb * 128 + r) * 16;
                        // A = [h 2^15 | h 2^9 | l 2^21],  B = [h 2^15 | l 2^21 | h 2^9]
                        *reinterpret_cast<uint4 *>(d0) = make_uint4(w15[0], w15[1], w15[2], w15[3]);
                        *reinterpret_cast<uint4 *>(d0 + PP_PART) =
                            isA ? make_uint4(w9[0], w9[1], w9[2], w9[3]) : make_uint4(wlo[0], wlo[1], wlo[2], wlo[3]);
                        *reinterpret_cast<uint4 *>(d0 + 2 * PP_PART) =
                            isA ? make_uint4(wlo[0], wlo[1], wlo[2], wlo[3]) : make_uint4(w9[0], w9[1], w9[2], w9[3]);
                    }
                    if (CULL && tid == 0) s_last[s] = (r0 >= n && k0 + PP_KC >= wlen) ? 1 : 0;
                    fence_proxy_async();  // this thread's generic-proxy stores -> visible to the tensor core
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&arrive_bar[s]);
                }
            }
            if (CULL && a.pairs && rank == 0 && tid == 0 && kept > 0) {  // cells of the pair tile x kept hits
                const int i0 = (c.t_m & ~1) * 128, j0 = c.t_n * TC_N;
                const long long cells = (long long)min(256, a.n0 - i0) * min(TC_N, a.n1 - j0);
                atomicAdd(a.pairs, (unsigned long long)(cells * kept));
            }
        }
    } else if (warp == PP_MMA_WARP) {
        // ------------------------------------------------------------------ MMA issuer (even CTA)
        if (rank == 1 && lane == 0) {
            // relay: once all 16 local warps have filled stage s, one release.cluster arrive on the
            // even CTA's full[s] publishes them (their stores precede their local arrivals, which
            // this thread acquires) -- one GPU-scope fence per chunk instead of sixteen
            const uint32_t full_addr0 = mapa_rank0(smem_u32(&s_full[0]));
            uint32_t cg = 0;
            for (int t = t0; t < t1; t += dt) {
                const PairCoord c = decode_pair(t, ppe, nl, tn, 1);
                const int n = a.offsets[c.e + 1] - a.offsets[c.e];
                int nck = 0;
                for (int w0 = 0; w0 < n; w0 += a.cap) nck += (min(a.cap, n - w0) + PP_KC - 1) / PP_KC;
                for (int ck = 0; CULL ? (n > 0) : (ck < nck); ++ck) {
                    const int s = (int)(cg % PP_NS);
                    mbar_wait(&s_pfull[s], (cg / PP_NS) & 1u);
                    const bool last = CULL && s_last[s];
                    mbar_arrive_remote(full_addr0 + (uint32_t)(s * sizeof(uint64_t)));
                    ++cg;
                    if (last) break;
                }
            }
        }
        if (rank == 0) {  // the whole warp runs the loop; elect.sync picks the issuing lane
            uint32_t cg = 0;
            int ti = 0;
            const uint32_t peer_acc_full = mapa_rank(smem_u32(&s_acc_full[0]), 1);
            for (int t = t0; t < t1; t += dt, ++ti) {
                const PairCoord c = decode_pair(t, ppe, nl, tn, 0);
                const int n = a.offsets[c.e + 1] - a.offsets[c.e];
                const int b = ti & 1;
                if (ti >= 2) mbar_wait_cluster(&s_acc_empty[b], ((ti >> 1) - 1) & 1);  // both epilogues done
                tc_fence_after();
                const uint32_t acc = tmem + (uint32_t)(b * TC_N);
                int nck = 0;  // chunks of this tile: every window is cut into 64-hit chunks
                for (int w0 = 0; w0 < n; w0 += a.cap) nck += (min(a.cap, n - w0) + PP_KC - 1) / PP_KC;
                bool last = false;  // CULL: the generating warps flag the tile's last chunk
                for (int ck = 0; CULL ? (n > 0 && !last) : (ck < nck); ++ck, ++cg) {
                    const int s = (int)(cg % PP_NS);
                    mbar_wait_cluster(&s_full[s], (cg / PP_NS) & 1u);
                    tc_fence_after();
                    if (CULL) last = s_last[s];
                    // descriptor of the stage's first A / B part; offsets inside the stage are added
                    // to the 14-bit start-address field (address >> 4) directly
                    const uint64_t dA = umma_desc(stage_saddr + s * PP_STAGE, 128 * 16, 128);
                    const uint64_t dB = dA + (uint64_t)((3 * PP_PART) >> 4);
#pragma unroll
                    for (int j = 0; j < PP_KC / 16; ++j) {  // K = 16 fp16 per MMA = 2 k-blocks
                        const uint32_t o = j * 2 * (128 * 16);
#pragma unroll
                        for (int pp = 0; pp < 3; ++pp)
                            tc2_mma_f16_warp(acc, dA + (uint64_t)((pp * PP_PART + o) >> 4),
                                             dB + (uint64_t)((pp * PP_PART + o) >> 4),
                                             (ck > 0 || j > 0 || pp > 0) ? 1u : 0u);
                    }
                    tc2_commit_both_warp(&s_empty[s]);
                }
                if (CULL ? n > 0 : nck > 0) {
                    tc2_commit_both_warp(&s_acc_full[b]);  // both CTAs: every MMA of this tile complete
                } else if (lane == 0) {
                    mbar_arrive(&s_acc_full[b]);
                    mbar_arrive_remote(peer_acc_full + (uint32_t)(b * sizeof(uint64_t)));
                }
                __syncwarp();
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------------ epilogue warps
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const uint32_t acc_empty0 = mapa_rank0(smem_u32(&s_acc_empty[0]));
        const int64_t cells = (int64_t)a.n0 * a.n1 * nl;
        int ti = 0;
        uint32_t epi_n = 0;  // TMA_EPI: boxes stored so far (two per warp alternate)
        for (int t = t0; t < t1; t += dt, ++ti) {
            const PairCoord c = decode_pair(t, ppe, nl, tn, (int)rank);
            const int n = a.offsets[c.e + 1] - a.offsets[c.e];
            const int b = ti & 1;
            mbar_wait(&s_acc_full[b], (ti >> 1) & 1);
            tc_fence_after();
            const int i = c.t_m * 128 + q * 32 + lane;
            float *out = a.R + (int64_t)(a.e_base + c.e) * cells + ((int64_t)c.l * a.n0 + i) * a.n1;
            const int plane = (a.e_base + c.e) * nl + c.l;  // [E][n2] planes of [n0][n1] (Z37)
            RETINA_ASSERT(c.l >= 0 && c.l < nl && c.t_m * 128 < a.n0 + 128 && c.t_n * TC_N < a.n1);
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
                if constexpr (TMA_EPI) {
                    // registers -> swizzled box in shared memory -> one TMA tensor store per warp
                    // (rows past n0 and columns past n1 are clipped by the tensor map's bounds)
                    const uint32_t box = smem_u32(s_epi) + (uint32_t)((q * 2 + (epi_n & 1)) * PP_EPI_BOX);
                    if (epi_n >= 2) {  // the store issued from this box two boxes ago has read it
                        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        __syncwarp();
                    }
                    const uint32_t row = box + (uint32_t)(lane * 64), sw = (uint32_t)((lane >> 1) & 3);
#pragma unroll
                    for (int x = 0; x < 4; ++x)
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + (((uint32_t)x ^ sw) << 4)),
                                     "r"(v[4 * x]), "r"(v[4 * x + 1]), "r"(v[4 * x + 2]), "r"(v[4 * x + 3])
                                     : "memory");
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        asm volatile(
                            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                                reinterpret_cast<uint64_t>(&out_map)),
                            "r"(box), "r"(j0), "r"(c.t_m * 128 + q * 32), "r"(plane)
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    ++epi_n;
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
            if (lane == 0) mbar_arrive_remote(acc_empty0 + (uint32_t)(b * sizeof(uint64_t)));
        }
        if (TMA_EPI && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores done
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();  // both CTAs are done with TMEM before the pair deallocates
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * TC_N));
    }
}

static int sm_count() {  // of the current device (a cheap attribute query, legal during graph capture)
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) !=
                                                  cudaSuccess || v <= 0)
        return 148;
    return v;
}

// The output as a 3-D tensor map {n1, n0, planes} (planes = events x z0 nodes) with 16 x 32 x 1
// boxes, 64-byte swizzle; false if the driver's encoder is unavailable or the layout does not
// qualify (row pitch n1 * 4 bytes must be a multiple of 16) -- then the epilogue stores directly.
static bool encode_out_map(CUtensorMap *map, float *R, int n0, int n1, long long planes) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode || (n1 & 3) || (reinterpret_cast<uintptr_t>(R) & 15u) || planes <= 0) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)n1, (cuuint64_t)n0, (cuuint64_t)planes};
    const cuuint64_t strides[2] = {(cuuint64_t)n1 * 4, (cuuint64_t)n1 * n0 * 4};
    const cuuint32_t box[3] = {16, 32, 1}, estr[3] = {1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, R, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODEL, bool ZREF, bool TMA_EPI, bool CULL = false>
static cudaError_t launch_pp(const GridArgs &a0, int n_events, const CUtensorMap &map, cudaStream_t stream) {
    auto kern = grid_tensor16pp_kernel<MODEL, ZREF, TMA_EPI, CULL>;
    GridArgs a = a0;
    // hit window: x, y, z (+ the low part of z - z_ref) as floats; whole chunks
    constexpr int n_arr = (ZREF || MODEL == kSlope3) ? 4 : 3;
    constexpr int fixed = PP_NS * PP_STAGE + (TMA_EPI ? PP_EPI_BYTES : 0);
    const int cap_max = (227 * 1024 - fixed - 2048) / (4 * n_arr);
    a.cap = std::max(PP_KC, (std::min(std::max(a.cap, PP_KC), cap_max) / PP_KC) * PP_KC);
    const size_t smem = (size_t)fixed + (size_t)a.cap * 4 * n_arr;
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const long long per_event =
        (long long)((a0.n0 + 255) / 256) * ((a0.n1 + TC_N - 1) / TC_N) * (MODEL == kSlope3 ? a0.n2 : 1);
    const int ev_per_launch = (int)std::max(1LL, std::min((long long)n_events, 0x7fffffffLL / per_event));
    for (int e0 = 0; e0 < n_events; e0 += ev_per_launch) {
        GridArgs b = a;
        const int ne = std::min(ev_per_launch, n_events - e0);
        b.offsets = a.offsets + e0;  // event e of this launch = e0 + e of the batch
        b.e_base = e0;
        const int items = (int)(per_event * ne);
        const int clusters = std::max(1, std::min(items, sm_count() / 2));
        kern<<<2 * clusters, 32 * PP_WARPS, smem, stream>>>(b, items, map);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

template <int MODEL, bool ZREF>
static cudaError_t launch_pp_any(const GridArgs &a, int n_events, bool cull, cudaStream_t stream) {
    CUtensorMap map;
    const long long planes = (long long)n_events * (MODEL == kSlope3 ? a.n2 : 1);
    if (encode_out_map(&map, a.R, a.n0, a.n1, planes))  // (culling rides on the TMA-store variant only)
        return cull ? launch_pp<MODEL, ZREF, true, true>(a, n_events, map, stream)
                    : launch_pp<MODEL, ZREF, true>(a, n_events, map, stream);
    memset(&map, 0, sizeof(map));
    return launch_pp<MODEL, ZREF, false>(a, n_events, map, stream);
}

cudaError_t launch_grid_tensor16p(int model, const GridArgs &a, int n_events, cudaStream_t stream, bool cull) {
    if (n_events == 0) return cudaSuccess;
    if (model == kSlope3) return launch_pp_any<kSlope3, false>(a, n_events, cull, stream);
    if (model != kSlope2) return cudaErrorInvalidValue;
    return (a.z_ref == 0.f) ? launch_pp_any<kSlope2, false>(a, n_events, cull, stream)
                            : launch_pp_any<kSlope2, true>(a, n_events, cull, stream);
}

}  // namespace retina
