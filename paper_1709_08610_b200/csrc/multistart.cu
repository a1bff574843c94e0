// multistart.cu -- K4: Algorithm 1's update loop with update = fixed-step
// gradient ascent clamped to the prior box (Z7):
//     theta^{j+1} = clamp(theta^j + step * grad R(theta^j)),  j < n_iters,
// then R(theta^n) and (optionally) grad R(theta^n).
//
// Mapping (K4): grid = (seed blocks, events), 128 threads per CTA, each thread
// owns S = 8 seeds (lanes over consecutive seeds: coalesced seed loads / stores).  The event's
// hits are staged ONCE in shared memory by a TMA bulk copy and stay resident for all
// n_iters + 1 passes when they fit (HitStage); otherwise they stream per pass.  SLOPE3 CTAs also
// build a table of the event's detector planes once and loop plane by plane; a dense SLOPE3
// event whose float4 stage would limit occupancy is staged as (x, y) pairs + that table.  Each
// pass accumulates, per seed, R = sum w and the raw gradient sums in registers, in hit-array
// order; the 2/sigma^2 factor is applied once per seed.  SLOPE3 forms its residuals already
// scaled by sqrt(K) (see ms_pass_x2), so its gradient factor is c2 / sqrt(K).
//
// Gradient (chain rule through s^2):
//   LINE2D  s = y - a x - b:           dR/da = c2 sum w s x,   dR/db = c2 sum w s
//   SLOPE2  s = (x - tx d, y - ty d):  dR/dtx = c2 sum w s_x d, dR/dty = c2 sum w s_y d
//   SLOPE3  d = z - z0:                ... and dR/dz0 = -c2 (tx sum w s_x + ty sum w s_y)
// with w = exp(-s^2/sigma^2) = ex2(-K s^2), c2 = 2/sigma^2.
#include "common.cuh"
#include "kernels.cuh"
#include "cull.cuh"

#include <algorithm>
#include <type_traits>

namespace retina {

#ifndef RETINA_MS_THREADS
#define RETINA_MS_THREADS 128
#endif
#ifndef RETINA_MS_MINB
#define RETINA_MS_MINB 6  // caps registers at 80: 6 CTAs (24 warps) per SM, measured +3 % over 94 registers
#endif
#ifndef RETINA_MS3_SEEDS  // SLOPE3 carries z0 and the exact d = z - z0 per seed: fewer seeds per thread
#define RETINA_MS3_SEEDS 4
#endif
#ifndef RETINA_MS3_MINB
#define RETINA_MS3_MINB 6
#endif
constexpr int kMsThreads = RETINA_MS_THREADS;

template <int MODEL, int S, bool ZREF, bool GRAD>
__device__ __forceinline__ void ms_pass(HitStage &st, const float (&th)[S][3], float negK, float zref,
                                        float (&R)[S], float (&G)[S][4]) {
    // G[s][0..1]: sum w s_x d, sum w s_y d;  G[s][2..3] (SLOPE3): sum w s_x, sum w s_y.
    // SLOPE2/3 gradients are accumulated per detector plane (hits with equal z, which are
    // contiguous when hits are sorted by z): Q = sum_{k in plane} w s, then G += d_plane Q at
    // each plane change.  This saves the per-pair w*d multiply (the FMA pipe is the binding
    // unit of this loop); unsorted hits only make planes shorter, never wrong.
#pragma unroll
    for (int s = 0; s < S; ++s) {
        R[s] = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) G[s][i] = 0.f;
    }
    float dh[S], dl[S], qx[S], qy[S];
#pragma unroll
    for (int s = 0; s < S; ++s) dh[s] = dl[s] = qx[s] = qy[s] = 0.f;
    float zprev = __int_as_float(0x7fc00000);  // NaN: the first hit always opens a plane
    float dprev = 0.f, dlprev = 0.f;           // SLOPE2: d of the open plane (hi, lo)
    auto flush = [&]() {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const float d = (MODEL == kSlope3) ? dh[s] : dprev;
            G[s][0] = __fmaf_rn(d, qx[s], G[s][0]);
            G[s][1] = __fmaf_rn(d, qy[s], G[s][1]);
            if (MODEL == kSlope3) {
                G[s][2] = __fadd_rn(G[s][2], qx[s]);
                G[s][3] = __fadd_rn(G[s][3], qy[s]);
            }
            qx[s] = qy[s] = 0.f;
        }
    };
    st.pass([&](const float4 *h, int len) {
#pragma unroll 2
        for (int k = 0; k < len; ++k) {
            const float4 hk = h[k];
            if (MODEL == kSlope2) {
                if (hk.z != zprev) {  // warp-uniform: every thread reads the same hit
                    if (GRAD) flush();
                    zprev = hk.z;
                    if (ZREF)
                        two_sum(hk.z, -zref, dprev, dlprev);
                    else
                        dprev = hk.z;
                }
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    float sx, sy;
                    if (ZREF) {
                        sx = __fmaf_rn(-th[s][0], dlprev, __fmaf_rn(-th[s][0], dprev, hk.x));
                        sy = __fmaf_rn(-th[s][1], dlprev, __fmaf_rn(-th[s][1], dprev, hk.y));
                    } else {
                        sx = __fmaf_rn(-th[s][0], hk.z, hk.x);
                        sy = __fmaf_rn(-th[s][1], hk.z, hk.y);
                    }
                    const float q = __fmaf_rn(sx, sx, __fmul_rn(sy, sy));
                    const float w = ex2_approx(__fmul_rn(q, negK));
                    R[s] = __fadd_rn(R[s], w);
                    if (GRAD) {
                        qx[s] = __fmaf_rn(w, sx, qx[s]);
                        qy[s] = __fmaf_rn(w, sy, qy[s]);
                    }
                }
            } else if (MODEL == kSlope3) {
                if (hk.z != zprev) {
                    if (GRAD) flush();
                    zprev = hk.z;
#pragma unroll
                    for (int s = 0; s < S; ++s) two_sum(hk.z, -th[s][2], dh[s], dl[s]);
                }
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const float sx = __fmaf_rn(-th[s][0], dl[s], __fmaf_rn(-th[s][0], dh[s], hk.x));
                    const float sy = __fmaf_rn(-th[s][1], dl[s], __fmaf_rn(-th[s][1], dh[s], hk.y));
                    const float q = __fmaf_rn(sx, sx, __fmul_rn(sy, sy));
                    const float w = ex2_approx(__fmul_rn(q, negK));
                    R[s] = __fadd_rn(R[s], w);
                    if (GRAD) {
                        qx[s] = __fmaf_rn(w, sx, qx[s]);
                        qy[s] = __fmaf_rn(w, sy, qy[s]);
                    }
                }
            } else {  // LINE2D
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const float p_hi = __fmul_rn(th[s][0], hk.x);
                    const float p_lo = __fmaf_rn(th[s][0], hk.x, -p_hi);
                    float r_hi, e1;
                    two_sum(hk.y, -p_hi, r_hi, e1);
                    const float sres = __fadd_rn(__fsub_rn(r_hi, th[s][1]), __fsub_rn(e1, p_lo));
                    const float w = ex2_approx(__fmul_rn(__fmul_rn(sres, sres), negK));
                    R[s] = __fadd_rn(R[s], w);
                    if (GRAD) {
                        const float ws = __fmul_rn(w, sres);
                        G[s][0] = __fmaf_rn(ws, hk.x, G[s][0]);
                        G[s][1] = __fadd_rn(G[s][1], ws);
                    }
                }
            }
        }
    });
    if (GRAD && MODEL != kLine2D) flush();
}

// SLOPE2 / SLOPE3 pass on seed PAIRS with packed f32x2 arithmetic (FFMA2 / FMUL2 / FADD2):
// every instruction of the per-pair chain serves two seeds, halving issue slots.  Each half
// is an independent IEEE round-to-nearest operation, so results are bit-identical to the
// scalar ms_pass.  Per (seed, hit): 8 FMA-pipe lane-ops + 1 MUFU.EX2, i.e. the loop is
// balanced between the FMA pipe (128 lanes/clk/SM) and MUFU (16/clk/SM).
// Detector planes of a resident event (hits sorted by z: runs of equal z), built once per CTA so
// the passes loop plane by plane instead of testing every hit for a plane change.
constexpr int kMaxPlanes = 64;
struct PlaneTable {
    const int *start;  // [np + 1]
    const float *z;    // [np]
    int np;            // -1: no table (streaming event, or more than kMaxPlanes runs)
    const float2 *xy;  // compact stage: (x, y) per hit (z from the table); nullptr: float4 hits
};

// Compact stage (dense SLOPE3 events, whose float4 stage would leave too few CTAs per SM): every
// thread converts hits to (x, y) pairs in shared memory (8 B instead of 16 per hit), and the warps
// list the plane starts in order from the z values in global memory (each warp a contiguous run
// of hits, then a prefix over the warps).  np = -1 when there are more than kMaxPlanes planes.
__device__ __forceinline__ PlaneTable build_compact(const float4 *__restrict__ gh, int n, float2 *s_xy,
                                                    int *s_start, float *s_z, int *s_np, int *s_wcnt) {
    const int nw = blockDim.x >> 5, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const float4 h = __ldg(gh + k);
        s_xy[k] = make_float2(h.x, h.y);
    }
    const int seg = (n + nw - 1) / nw, a = min(n, w * seg), b = min(n, a + seg);
    auto flag = [&](int k) { return k < b && (k == 0 || !(__ldg(&gh[k].z) == __ldg(&gh[k - 1].z))); };
    int cnt = 0;
    for (int base = a; base < b; base += 32) cnt += __popc(__ballot_sync(0xffffffffu, flag(base + lane)));
    if (lane == 0) s_wcnt[w] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int i = 0; i < nw; ++i) {
            const int c = s_wcnt[i];
            s_wcnt[i] = acc;
            acc += c;
        }
        s_start[min(acc, kMaxPlanes)] = n;
        *s_np = (acc <= kMaxPlanes) ? acc : -1;
    }
    __syncthreads();
    int off = s_wcnt[w];
    for (int base = a; base < b; base += 32) {
        const int k = base + lane;
        const bool f = flag(k);
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        const int pos = off + __popc(bal & ((1u << lane) - 1u));
        if (f && pos < kMaxPlanes) {
            s_start[pos] = k;
            s_z[pos] = __ldg(&gh[k].z);
        }
        off += __popc(bal);
    }
    __syncthreads();
    return PlaneTable{s_start, s_z, *s_np, s_xy};
}

// warp 0 lists the starts of the runs of equal z in order; every thread returns the table
__device__ __forceinline__ PlaneTable build_planes(const float4 *h, int n, int *s_start, float *s_z, int *s_np) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        int cnt = 0;
        for (int base = 0; base < n; base += 32) {
            const int k = base + lane;
            const bool f = k < n && (k == 0 || !(h[k].z == h[k - 1].z));
            const unsigned b = __ballot_sync(0xffffffffu, f);
            const int pos = cnt + __popc(b & ((1u << lane) - 1u));
            if (f && pos < kMaxPlanes) {
                s_start[pos] = k;
                s_z[pos] = h[k].z;
            }
            cnt += __popc(b);
        }
        if (lane == 0) {
            s_start[min(cnt, kMaxPlanes)] = n;
            *s_np = (cnt <= kMaxPlanes) ? cnt : -1;
        }
    }
    __syncthreads();
    return PlaneTable{s_start, s_z, *s_np, nullptr};
}

#ifndef RETINA_MC_BATCH
#define RETINA_MC_BATCH 1  // K4c list loop: 4 listed hits per step (0: one at a time; 8 per step measured no faster)
#endif
// list != nullptr (K4c): only the resident hits list[0 .. L) are visited, in that (hit) order; a
// new plane is found by comparing z, which runs the same operations as the plane table would.
template <int MODEL, int S, bool ZREF, bool GRAD, bool WANT_R>
__device__ __forceinline__ void ms_pass_x2(HitStage &st, const float (&th)[S][3], float negK, float zref,
                                           float (&R)[S], float (&G)[S][4], float sk, const PlaneTable &pt,
                                           const uint16_t *list = nullptr, int L = 0) {
    static_assert(S % 2 == 0, "seed pairs");
    constexpr int NP = S / 2;
    float2 mtx[NP], mty[NP], r2[NP], qx[NP], qy[NP], gx[NP], gy[NP], ax[NP], ay[NP], dh[NP], dl[NP];
    const float2 zero = make_float2(0.f, 0.f);
    // SLOPE3, per plane and seed: c = t (z - z0) as chx + clx (clx ~ 1e-5 of an ulp-level tail), and
    // the tail pre-scaled by -sk; per hit s' = sk s = fma(sk, x - chx, -sk clx): x - chx is exact for
    // every hit near the track (Sterbenz) and one rounding relative to |s| otherwise, and the scale
    // rides on the correction FMA, so a = s'_x^2 + s'_y^2 needs no separate multiply by K
    float2 chx[NP], chy[NP], cx[NP], cy[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) chx[p] = chy[p] = cx[p] = cy[p] = zero;
    const float2 SK = make_float2(sk, sk);
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        mtx[p] = make_float2(-th[2 * p][0], -th[2 * p + 1][0]);
        mty[p] = make_float2(-th[2 * p][1], -th[2 * p + 1][1]);
        r2[p] = qx[p] = qy[p] = gx[p] = gy[p] = ax[p] = ay[p] = dh[p] = dl[p] = zero;
    }
    const float2 nk = make_float2(negK, negK);
    float zprev = __int_as_float(0x7fc00000);
    float dprev = 0.f, dlprev = 0.f;
    auto flush = [&]() {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float2 d = (MODEL == kSlope3) ? dh[p] : make_float2(dprev, dprev);
            gx[p] = __ffma2_rn(d, qx[p], gx[p]);
            gy[p] = __ffma2_rn(d, qy[p], gy[p]);
            if (MODEL == kSlope3) {
                ax[p] = __fadd2_rn(ax[p], qx[p]);
                ay[p] = __fadd2_rn(ay[p], qy[p]);
            }
            qx[p] = qy[p] = zero;
        }
    };
    // a new detector plane at z (the same operations, in the same order, whether found from the
    // table or by comparing a hit's z with the previous one)
    auto plane = [&](const float z) {
        if (GRAD) flush();
        zprev = z;
        {
            const float4 hk = make_float4(0.f, 0.f, z, 0.f);
            if (MODEL == kSlope3) {
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    two_sum(hk.z, -th[2 * p][2], dh[p].x, dl[p].x);
                    two_sum(hk.z, -th[2 * p + 1][2], dh[p].y, dl[p].y);
                    // t d = (t d_hi) + (t d_lo): ch = fl(t d_hi), its FMA residual + t d_lo as the tail
                    const float2 tx = make_float2(-mtx[p].x, -mtx[p].y), ty = make_float2(-mty[p].x, -mty[p].y);
                    chx[p] = __fmul2_rn(tx, dh[p]);
                    chy[p] = __fmul2_rn(ty, dh[p]);
                    const float2 lx = __ffma2_rn(tx, dl[p], __ffma2_rn(tx, dh[p], make_float2(-chx[p].x, -chx[p].y)));
                    const float2 ly = __ffma2_rn(ty, dl[p], __ffma2_rn(ty, dh[p], make_float2(-chy[p].x, -chy[p].y)));
                    cx[p] = __fmul2_rn(make_float2(-sk, -sk), lx);  // -sk x tail: constant over the plane
                    cy[p] = __fmul2_rn(make_float2(-sk, -sk), ly);
                }
            } else if (ZREF) {
                two_sum(hk.z, -zref, dprev, dlprev);
            } else {
                dprev = hk.z;
            }
        }
    };
    // one hit against every seed pair of the thread
    auto body = [&](const float4 hk) {
        const float2 X = make_float2(hk.x, hk.x), Y = make_float2(hk.y, hk.y);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float2 sx, sy;
            if (MODEL == kSlope3) {
                // scaled residuals s' = sk s (see the plane setup above)
                sx = __ffma2_rn(SK, __fadd2_rn(X, make_float2(-chx[p].x, -chx[p].y)), cx[p]);
                sy = __ffma2_rn(SK, __fadd2_rn(Y, make_float2(-chy[p].x, -chy[p].y)), cy[p]);
            } else if (ZREF) {
                const float2 D = make_float2(dprev, dprev), DL = make_float2(dlprev, dlprev);
                sx = __ffma2_rn(mtx[p], DL, __ffma2_rn(mtx[p], D, X));
                sy = __ffma2_rn(mty[p], DL, __ffma2_rn(mty[p], D, Y));
            } else {
                const float2 Z = make_float2(hk.z, hk.z);
                sx = __ffma2_rn(mtx[p], Z, X);
                sy = __ffma2_rn(mty[p], Z, Y);
            }
            float2 w;
            if (MODEL == kSlope3) {  // already scaled: 2^-(s'_x^2 + s'_y^2)
                const float2 a = __ffma2_rn(sx, sx, __fmul2_rn(sy, sy));
                w = make_float2(ex2_approx(-a.x), ex2_approx(-a.y));
            } else {
                const float2 a = __fmul2_rn(__ffma2_rn(sx, sx, __fmul2_rn(sy, sy)), nk);
                w = make_float2(ex2_approx(a.x), ex2_approx(a.y));
            }
            if (WANT_R) r2[p] = __fadd2_rn(r2[p], w);  // iterations only need grad R
            if (GRAD) {
                qx[p] = __ffma2_rn(w, sx, qx[p]);
                qy[p] = __ffma2_rn(w, sy, qy[p]);
            }
        }
    };
    if (list != nullptr) {  // K4c: the warp's listed hits
        const float4 *h = st.buf;
        auto one = [&](const float4 hk) {
            if (hk.z != zprev) plane(hk.z);  // warp-uniform: the list is the warp's
            body(hk);
        };
        int t = 0;
#if RETINA_MC_BATCH
        // four indices per 8-byte load, then four independent hit loads: no load waits on the
        // previous hit's index (the list is 16-byte aligned: cap % 8 == 0)
        for (; t + 4 <= L; t += 4) {
            const ushort4 ix = *reinterpret_cast<const ushort4 *>(list + t);
            const float4 h0 = h[ix.x], h1 = h[ix.y], h2 = h[ix.z], h3 = h[ix.w];
            one(h0);
            one(h1);
            one(h2);
            one(h3);
        }
#endif
#pragma unroll 2
        for (; t < L; ++t) one(h[list[t]]);
    } else if (pt.np >= 0 && pt.xy) {  // compact stage: (x, y) pairs, plane by plane
        for (int pl = 0; pl < pt.np; ++pl) {
            const int k1 = pt.start[pl + 1];
            plane(pt.z[pl]);
#pragma unroll 2
            for (int k = pt.start[pl]; k < k1; ++k) {
                const float2 q = pt.xy[k];
                body(make_float4(q.x, q.y, 0.f, 0.f));  // (SLOPE3's body reads x and y only)
            }
        }
    } else if (pt.np >= 0) {  // resident event: plane by plane
        const float4 *h = st.buf;
        for (int pl = 0; pl < pt.np; ++pl) {
            const int k1 = pt.start[pl + 1];
            plane(pt.z[pl]);
#pragma unroll 2
            for (int k = pt.start[pl]; k < k1; ++k) body(h[k]);
        }
    } else {
        st.pass([&](const float4 *h, int len) {
#pragma unroll 2
            for (int k = 0; k < len; ++k) {
                const float4 hk = h[k];
                if (hk.z != zprev) plane(hk.z);  // warp-uniform plane change
                body(hk);
            }
        });
    }
    if (GRAD) flush();
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        R[2 * p] = r2[p].x;
        R[2 * p + 1] = r2[p].y;
        G[2 * p][0] = gx[p].x;
        G[2 * p + 1][0] = gx[p].y;
        G[2 * p][1] = gy[p].x;
        G[2 * p + 1][1] = gy[p].y;
        G[2 * p][2] = ax[p].x;
        G[2 * p + 1][2] = ax[p].y;
        G[2 * p][3] = ay[p].x;
        G[2 * p + 1][3] = ay[p].y;
    }
}

template <int MODEL, int S, bool ZREF, bool GRAD, bool WANT_R>
__device__ __forceinline__ void ms_eval(HitStage &st, const float (&th)[S][3], float negK, float zref,
                                        float (&R)[S], float (&G)[S][4], float sk, const PlaneTable &pt) {
    if constexpr (MODEL == kLine2D)
        ms_pass<MODEL, S, ZREF, GRAD>(st, th, negK, zref, R, G);
    else
        ms_pass_x2<MODEL, S, ZREF, GRAD, WANT_R>(st, th, negK, zref, R, G, sk, pt);
}

template <int MODEL, int S>
__device__ __forceinline__ void ms_gradient(const float (&th)[S][3], const float (&G)[S][4], float c2,
                                            float (&g)[S][3]) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
        g[s][0] = __fmul_rn(c2, G[s][0]);
        g[s][1] = __fmul_rn(c2, G[s][1]);
        g[s][2] = (MODEL == kSlope3)
                      ? -__fmul_rn(c2, __fmaf_rn(th[s][0], G[s][2], __fmul_rn(th[s][1], G[s][3])))
                      : 0.f;
    }
}

// T threads per CTA (128 by default; 256 / 512 when an event's hits are so many that shared
// memory would otherwise cut the CTAs per SM below the 6 x 4 warps the register budget allows)
template <int MODEL, int S, bool ZREF, int T>
__global__ void __launch_bounds__(T, ((MODEL == kSlope3) ? RETINA_MS3_MINB : RETINA_MS_MINB) * kMsThreads / T)
multistart_kernel(MultistartArgs a) {
    extern __shared__ __align__(16) float4 s_hits[];
    __shared__ __align__(8) uint64_t s_bar[2];
    constexpr int P = (MODEL == kSlope3) ? 3 : 2;

    const int e = a.e_base + blockIdx.y;
    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;
    HitStage st;
    // compact SLOPE3 stage: a.cap float2 slots, i.e. a.cap / 2 float4 slots for the fallback stage
    st.init(s_hits, s_bar, a.hits + start, nh, (MODEL == kSlope3 && a.compact) ? a.cap / 2 : a.cap);
    __shared__ int s_pstart[kMaxPlanes + 1], s_np, s_wcnt[T / 32];
    __shared__ float s_pz[kMaxPlanes];
    PlaneTable pt{nullptr, nullptr, -1, nullptr};
    // SLOPE3 only: its plane change (two TwoSums and the scaled tails per seed pair) is the heavy
    // one; for SLOPE2 the per-hit test measured cheaper than the per-plane loop (cfg3 106.1 vs
    // 109.5 ms per 1000 events; cfg4 98.5 -> 97.1 ms per 200, cfg4 dense 115.7 -> 109.3 per 50)
    if (MODEL == kSlope3 && a.compact) {
        if (nh > 0 && nh <= a.cap)
            pt = build_compact(a.hits + start, nh, reinterpret_cast<float2 *>(s_hits), s_pstart, s_pz, &s_np, s_wcnt);
        if (pt.np < 0) pt = PlaneTable{nullptr, nullptr, -1, nullptr};  // too many planes: float4 stage streams
    } else if (MODEL == kSlope3 && st.load_resident()) {
        pt = build_planes(st.buf, nh, s_pstart, s_pz, &s_np);
    }

    int sid[S];
    float th[S][3];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        sid[s] = blockIdx.x * (T * S) + s * T + threadIdx.x;
        const int64_t src = ((int64_t)e * a.n_seeds + min(sid[s], a.n_seeds - 1)) * P;
#pragma unroll
        for (int i = 0; i < 3; ++i) th[s][i] = (i < P) ? __ldg(a.seeds + src + i) : 0.f;
    }

    float R[S], G[S][4], g[S][3];
    for (int it = 0; it < a.n_iters; ++it) {
        ms_eval<MODEL, S, ZREF, true, false>(st, th, a.negK, a.z_ref, R, G, a.sk, pt);
        ms_gradient<MODEL, S>(th, G, (MODEL == kSlope3) ? a.c2s : a.c2, g);
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int i = 0; i < P; ++i)
                th[s][i] = fminf(fmaxf(__fmaf_rn(a.step, g[s][i], th[s][i]), a.lo[i]), a.hi[i]);
    }
    if (a.grad_out) {
        ms_eval<MODEL, S, ZREF, true, true>(st, th, a.negK, a.z_ref, R, G, a.sk, pt);
        ms_gradient<MODEL, S>(th, G, (MODEL == kSlope3) ? a.c2s : a.c2, g);
    } else {
        ms_eval<MODEL, S, ZREF, false, true>(st, th, a.negK, a.z_ref, R, G, a.sk, pt);
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (sid[s] < a.n_seeds) {
            const int64_t o = (int64_t)e * a.n_seeds + sid[s];
            a.R_out[o] = R[s];
#pragma unroll
            for (int i = 0; i < P; ++i) {
                a.theta_out[o * P + i] = th[s][i];
                if (a.grad_out) a.grad_out[o * P + i] = g[s][i];
            }
        }
    }
}

#ifndef RETINA_MS_SEEDS
#define RETINA_MS_SEEDS 8
#endif
template <int MODEL, bool ZREF, int T>
static cudaError_t launch_ms_t(const MultistartArgs &a0, int n_events, cudaStream_t stream) {
    constexpr int S = (MODEL == kSlope3) ? RETINA_MS3_SEEDS : RETINA_MS_SEEDS;
    auto kern = multistart_kernel<MODEL, S, ZREF, T>;
    const size_t smem = (size_t)a0.cap * (a0.compact ? sizeof(float2) : sizeof(float4));
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const int blocks = (a0.n_seeds + T * S - 1) / (T * S);
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        MultistartArgs a = a0;
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        kern<<<dim3(blocks, ne), T, smem, stream>>>(a);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

template <int MODEL, bool ZREF>
static cudaError_t launch_ms(const MultistartArgs &a0, int n_events, cudaStream_t stream) {
    MultistartArgs a = a0;
    const int want = (MODEL == kSlope3) ? RETINA_MS3_MINB : RETINA_MS_MINB;
    // resident 128-thread CTAs the hit stage allows per SM (227 KB of shared memory); a SLOPE3
    // stage that would allow fewer than `want` is staged compactly ((x, y) + plane table, 8 B/hit)
    a.compact = (MODEL == kSlope3 && (int)((227 * 1024) / ((size_t)a.cap * sizeof(float4) + 1024)) < want) ? 1 : 0;
    const size_t per_cta = (size_t)a.cap * (a.compact ? sizeof(float2) : sizeof(float4)) + 1024;
    const int fit = (int)((227 * 1024) / per_cta);
    if constexpr (MODEL == kLine2D) {  // (2-D toy events: always small)
        return launch_ms_t<MODEL, ZREF, kMsThreads>(a, n_events, stream);
    } else {
        if (fit >= want) return launch_ms_t<MODEL, ZREF, kMsThreads>(a, n_events, stream);
        if (2 * fit >= want) return launch_ms_t<MODEL, ZREF, 2 * kMsThreads>(a, n_events, stream);
        return launch_ms_t<MODEL, ZREF, 4 * kMsThreads>(a, n_events, stream);
    }
}

cudaError_t launch_multistart(int model, const MultistartArgs &a, int n_events, cudaStream_t stream) {
    if (n_events == 0 || a.n_seeds == 0) return cudaSuccess;
    switch (model) {
        case kLine2D: return launch_ms<kLine2D, false>(a, n_events, stream);
        case kSlope2:
            return (a.z_ref == 0.f) ? launch_ms<kSlope2, false>(a, n_events, stream)
                                    : launch_ms<kSlope2, true>(a, n_events, stream);
        case kSlope3: return launch_ms<kSlope3, false>(a, n_events, stream);
    }
    return cudaErrorInvalidValue;
}

// =====================================================================================================
// K4c: the SLOPE2 multi-start update loop of K4 (Algorithm 1 update loop,
// PAPER.md:144-153; Z7) computing the SAME results bit for bit while evaluating only the
// (seed, hit) pairs that can contribute.
//
// Why it is exact: w = ex2.approx.ftz(-K s^2) is +0 whenever -K s^2 < -126 (the result would be
// subnormal and is flushed), and adding w = +0 to R, or w * s_x = +-0 to the gradient sums, leaves
// them unchanged (the sums never hold -0: they start at +0 and -0 + +0 = +0).  A hit is skipped by a
// warp only when a conservative bound proves K s^2 > 128 for EVERY seed of the warp; the warp then
// visits the remaining hits in the original hit order with the same operations as K4 (FFMA2 seed
// pairs, per-plane gradient sums flushed at each change of z), so every sum sees the same non-zero
// terms in the same order.
//
// Where the speed comes from: seeds are first ordered per event along a Morton curve of (tx, ty)
// (K4c-sort, one CTA per event; the outputs go back to the caller's seed order), so the 256 seeds of
// a warp (8 per lane) cover a small box of parameter space.  Per iteration each warp reduces its box,
// lists (ballot, in order) the hits within reach of the box -- on cfg3 about one hit in ten -- and
// evaluates only those.  The work actually done is counted (pairs_evaluated).
#ifndef RETINA_MC_MINB
#define RETINA_MC_MINB 5  // CTAs per SM the register budget allows (96 registers: no spills)
#endif
#ifndef RETINA_MC_MARGIN
#define RETINA_MC_MARGIN 0.02f  // list box margin, relative to the seeds' box
#endif
#ifndef RETINA_MC_MARGIN_ABS
#define RETINA_MC_MARGIN_ABS 1e-5f
#endif
#ifndef RETINA_MC_UNITS
#define RETINA_MC_UNITS 16  // at most this many units of 256 seeds per block, dealt to its 4 warps
#endif
#ifndef RETINA_MC_SEEDS
#define RETINA_MC_SEEDS 2  // SLOPE2 seeds per thread in K4c (a unit = 32 x this: small units, tight boxes; 8 / 4 / 2 measured 31.2 / 22.8 / 17.0 ms per 2,000 cfg3 events)
#endif
#ifndef RETINA_MC3_SEEDS
#define RETINA_MC3_SEEDS 4  // SLOPE3 (4 / 2: 39.3 / 37.7 ms per 100 cfg4 events, but 278 / 295 ms on the full 1,000)
#endif
constexpr int kMcThreads = 128, kMcSeeds = RETINA_MC_SEEDS, kMcWarps = kMcThreads / 32, kMcUnits = RETINA_MC_UNITS;

// ---------------------------------------------------------------- K4c-sort: Morton order per event
// perm[e][q] = caller index of the q-th seed of event e along a Morton curve of the seed's
// parameters quantised over the prior box (P = 2: 16 bits per axis; P = 3: 10).  Bitonic sort of
// 32-bit keys -- the Morton code's leading 32 - ib bits, then the index (ib bits, N = 2^ib >= n,
// N >= 1024) -- with E = N / 1024 keys per thread in registers: compare-exchange stages of stride
// < E run inside a thread, strides < 32 E through warp shuffles, only the wider ones through
// shared memory (two block barriers each: 15 such stages for N = 8192 instead of 91 in a plain
// shared-memory network).  Any order gives the same results (it only groups seeds into warps);
// this one is deterministic.
__device__ __forceinline__ uint32_t morton_spread2(uint32_t x) {  // 16 bits -> even bit positions
    x &= 0xffffu;
    x = (x | (x << 8)) & 0x00ff00ffu;
    x = (x | (x << 4)) & 0x0f0f0f0fu;
    x = (x | (x << 2)) & 0x33333333u;
    return (x | (x << 1)) & 0x55555555u;
}
__device__ __forceinline__ uint32_t morton_spread3(uint32_t x) {  // 10 bits -> every third bit
    x &= 0x3ffu;
    x = (x | (x << 16)) & 0xff0000ffu;
    x = (x | (x << 8)) & 0x0300f00fu;
    x = (x | (x << 4)) & 0x030c30c3u;
    return (x | (x << 2)) & 0x09249249u;
}

// compare-exchange of register pairs (r, r ^ ST) of thread t's E consecutive keys
template <int E, int ST>
__device__ __forceinline__ void sort_cx_reg(uint32_t (&k)[E], int t, int size) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
        if ((r ^ ST) > r) {
            const bool up = ((t * E + r) & size) == 0;
            const uint32_t a = k[r], b = k[r ^ ST];
            k[r] = up ? min(a, b) : max(a, b);
            k[r ^ ST] = up ? max(a, b) : min(a, b);
        }
    }
}

template <int E>
__global__ void __launch_bounds__(1024) seed_morton_sort_kernel(const float *seeds, int n_seeds, int P, float3 lo,
                                                                float3 hi, int32_t *perm, int e_base) {
    constexpr int N = 1024 * E;
    constexpr int ib = 10 + (E >= 2) + (E >= 4) + (E >= 8) + (E >= 16);  // log2(N)
    extern __shared__ uint32_t s_key[];  // N + N / 32 words (one pad word per 32: no bank conflicts)
    const int e = e_base + blockIdx.x, t = threadIdx.x;
    const float *sd = seeds + (int64_t)e * n_seeds * P;
    const int bits = (P == 3) ? 10 : 16;
    const int mbits = P * bits, keep = 32 - ib;
    const float qmax = (float)((1 << bits) - 1);
    const float sc[3] = {qmax / fmaxf(hi.x - lo.x, 1e-30f), qmax / fmaxf(hi.y - lo.y, 1e-30f),
                         qmax / fmaxf(hi.z - lo.z, 1e-30f)};
    const float lo3[3] = {lo.x, lo.y, lo.z};
    uint32_t k[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int i = t * E + r;
        k[r] = 0xffffffffu;  // padding sorts last (a real key's index bits are < n - 1 < N - 1)
        if (i < n_seeds) {
            uint32_t m = 0;
            for (int d = 0; d < P; ++d) {
                const uint32_t q = (uint32_t)fminf(fmaxf((sd[(int64_t)P * i + d] - lo3[d]) * sc[d], 0.f), qmax);
                m |= (P == 3 ? morton_spread3(q) : morton_spread2(q)) << d;
            }
            const uint32_t top = (keep >= mbits) ? m : (m >> (mbits - keep));
            k[r] = (top << ib) | (uint32_t)i;
        }
    }
    auto pad = [](int i) { return i + (i >> 5); };
    for (int size = 2; size <= N; size <<= 1)
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            if (stride < E) {  // both elements in this thread (compile-time register indices)
                if (stride == 1) sort_cx_reg<E, 1>(k, t, size);
                if constexpr (E > 2) if (stride == 2) sort_cx_reg<E, 2>(k, t, size);
                if constexpr (E > 4) if (stride == 4) sort_cx_reg<E, 4>(k, t, size);
                if constexpr (E > 8) if (stride == 8) sort_cx_reg<E, 8>(k, t, size);
            } else if (stride < 32 * E) {  // partner in lane ^ (stride / E), same register
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const int i = t * E + r;
                    const uint32_t v = __shfl_xor_sync(0xffffffffu, k[r], stride / E);
                    const bool keep_min = ((i & stride) == 0) == ((i & size) == 0);
                    k[r] = keep_min ? min(k[r], v) : max(k[r], v);
                }
            } else {  // partner in another warp
#pragma unroll
                for (int r = 0; r < E; ++r) s_key[pad(t * E + r)] = k[r];
                __syncthreads();
#pragma unroll
                for (int r = 0; r < E; ++r) {
                    const int i = t * E + r;
                    const uint32_t v = s_key[pad(i ^ stride)];
                    const bool keep_min = ((i & stride) == 0) == ((i & size) == 0);
                    k[r] = keep_min ? min(k[r], v) : max(k[r], v);
                }
                __syncthreads();
            }
        }
    const uint32_t imask = (1u << ib) - 1u;
#pragma unroll
    for (int r = 0; r < E; ++r) {
        const int i = t * E + r;
        if (i < n_seeds) perm[(int64_t)e * n_seeds + i] = (int32_t)(k[r] & imask);
    }
}

// ---------------------------------------------------------------- K4c (box bound and lists: cull.cuh)
template <int MODEL, int S, bool ZREF>
__global__ void __launch_bounds__(kMcThreads, RETINA_MC_MINB)
    multistart_culled_kernel(MultistartArgs a, const int32_t *perm, unsigned long long *pairs_evaluated,
                             int units_per_cta) {
    constexpr int P = (MODEL == kSlope3) ? 3 : 2;
    constexpr int USEEDS = 32 * S;  // seeds per unit (one warp's)
    extern __shared__ __align__(16) float4 s_hits[];  // [cap] hits, then [warps][cap] uint16 lists
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ int s_next;
    const int e = a.e_base + blockIdx.y;
    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_next = 0;
    HitStage st;
    st.init(s_hits, s_bar, a.hits + start, nh, a.cap);  // (its block barrier also publishes s_next)
    // an event larger than the stage (max_event_hits is only a hint) runs K4's dense passes, streamed
    const bool culled = nh <= a.cap && nh <= 65535 && (nh == 0 || st.load_resident());
    uint16_t *list = reinterpret_cast<uint16_t *>(s_hits + a.cap) + warp * a.cap;
    const float K = -a.negK;
    const PlaneTable no_table{nullptr, nullptr, -1, nullptr};

    // Units of USEEDS seeds are dealt to the warps: dynamically (a shared counter) when the event is
    // resident -- the warps' lists differ in length, so a fixed share would leave warps idle -- and
    // round-robin in lockstep otherwise (the streamed dense passes synchronise the block).
    const int32_t *pe = perm + (int64_t)e * a.n_seeds;
    const int cta_seed0 = blockIdx.x * units_per_cta * USEEDS;
    const int units = min(units_per_cta, (a.n_seeds - cta_seed0 + USEEDS - 1) / USEEDS);
    unsigned long long evaluated = 0;
    for (int k = 0;; ++k) {
        int u;
        if (culled) {
            if (lane == 0) u = atomicAdd(&s_next, 1);
            u = __shfl_sync(0xffffffffu, u, 0);
            if (u >= units) break;
        } else {
            u = warp + kMcWarps * k;
            if (k >= (units + kMcWarps - 1) / kMcWarps) break;
        }
        // a unit = USEEDS consecutive seeds of the Morton order (S per lane, 32 consecutive per s)
        const int q0 = cta_seed0 + u * USEEDS + lane;
        bool ok[S];
        float th[S][3];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int q = q0 + s * 32;
            ok[s] = q < a.n_seeds;
            const int qo = __ldg(pe + min(q, a.n_seeds - 1));
            RETINA_ASSERT(qo >= 0 && qo < a.n_seeds);
            const int64_t src = ((int64_t)e * a.n_seeds + qo) * P;
#pragma unroll
            for (int i = 0; i < 3; ++i) th[s][i] = (i < P) ? __ldg(a.seeds + src + i) : 0.f;
        }
        int nvalid = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) nvalid += ok[s] ? 1 : 0;
        nvalid = __reduce_add_sync(0xffffffffu, nvalid);
        // The list is built for the seeds' box grown by a margin and rebuilt only when a seed leaves
        // that box (a list built for a box covers every seed inside it, so reuse stays exact); fixed-
        // step seeds move little per iteration.
        McBox lb;
        lb.lo[0] = 1.f;
        lb.hi[0] = 0.f;  // empty: build on the first pass
        int L = 0;

        float R[S], G[S][4], g[S][3];
        auto pass = [&](auto grad_tag, auto want_r_tag) {  // one pass over the hits in reach, or all of them
            constexpr bool GR = decltype(grad_tag)::value, WR = decltype(want_r_tag)::value;
            if (culled) {
                const McBox B = mc_warp_box<P, S>(th, ok);
                bool inside = lb.lo[0] <= lb.hi[0];
#pragma unroll
                for (int i = 0; i < P; ++i) inside = inside && B.lo[i] >= lb.lo[i] && B.hi[i] <= lb.hi[i];
                if (!inside) {
                    lb = B;
                    if (B.lo[0] <= B.hi[0])
#pragma unroll
                        for (int i = 0; i < P; ++i) {
                            const float m = fmaxf(RETINA_MC_MARGIN_ABS * (i == 2 ? 1e4f : 1.f),
                                                  RETINA_MC_MARGIN * (B.hi[i] - B.lo[i]));
                            lb.lo[i] = B.lo[i] - m;
                            lb.hi[i] = B.hi[i] + m;
                        }
                    L = mc_build_list<MODEL, ZREF>(st.buf, nh, lb, K, a.z_ref, list);
                }
                evaluated += (unsigned long long)L * nvalid;
                ms_pass_x2<MODEL, S, ZREF, GR, WR>(st, th, a.negK, a.z_ref, R, G, a.sk, no_table, list, L);
            } else {
                ms_eval<MODEL, S, ZREF, GR, WR>(st, th, a.negK, a.z_ref, R, G, a.sk, no_table);
                evaluated += (unsigned long long)nh * nvalid;
            }
        };
        const float cg = (MODEL == kSlope3) ? a.c2s : a.c2;
        for (int it = 0; it < a.n_iters; ++it) {
            pass(std::true_type{}, std::false_type{});
            ms_gradient<MODEL, S>(th, G, cg, g);
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int i = 0; i < P; ++i)
                    th[s][i] = fminf(fmaxf(__fmaf_rn(a.step, g[s][i], th[s][i]), a.lo[i]), a.hi[i]);
        }
        if (a.grad_out) {
            pass(std::true_type{}, std::true_type{});
            ms_gradient<MODEL, S>(th, G, cg, g);
        } else {
            pass(std::false_type{}, std::true_type{});
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!ok[s]) continue;
            const int64_t o = (int64_t)e * a.n_seeds + __ldg(pe + q0 + s * 32);
            a.R_out[o] = R[s];
#pragma unroll
            for (int i = 0; i < P; ++i) {
                a.theta_out[o * P + i] = th[s][i];
                if (a.grad_out) a.grad_out[o * P + i] = g[s][i];
            }
        }
    }
    if (pairs_evaluated && lane == 0 && evaluated) atomicAdd(pairs_evaluated, evaluated);
}

size_t multistart_culled_workspace_bytes(long long n_events, int n_seeds) {
    return (size_t)(n_events * n_seeds) * sizeof(int32_t);
}

bool multistart_culled_ok(int model, int n_seeds) {
    // SLOPE2 / SLOPE3; the sort holds an event's seeds in shared memory
    int np2 = 1;
    while (np2 < n_seeds) np2 <<= 1;
    return (model == kSlope2 || model == kSlope3) && n_seeds > 0 && np2 <= 16384;  // 64 KB of 32-bit keys
}

template <int E>
static cudaError_t launch_sort_e(const float *seeds, int n_seeds, int P, float3 lo, float3 hi, int32_t *perm,
                                 int n_events, cudaStream_t stream) {
    const size_t smem = (size_t)(1024 * E + 32 * E) * sizeof(uint32_t);
    cudaError_t err = ensure_dynamic_smem(seed_morton_sort_kernel<E>, smem);
    if (err != cudaSuccess) return err;
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        const int ne = std::min(65535, n_events - e0);
        seed_morton_sort_kernel<E><<<ne, 1024, smem, stream>>>(seeds, n_seeds, P, lo, hi, perm, e0);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

cudaError_t launch_seed_morton_sort(const float *seeds, int n_seeds, int P, const float (&lo)[3], const float (&hi)[3],
                                    int32_t *perm, int n_events, cudaStream_t stream) {
    int np2 = 1024;
    while (np2 < n_seeds) np2 <<= 1;
    const float3 l3 = make_float3(lo[0], lo[1], lo[2]), h3 = make_float3(hi[0], hi[1], hi[2]);
    switch (np2 / 1024) {
        case 1: return launch_sort_e<1>(seeds, n_seeds, P, l3, h3, perm, n_events, stream);
        case 2: return launch_sort_e<2>(seeds, n_seeds, P, l3, h3, perm, n_events, stream);
        case 4: return launch_sort_e<4>(seeds, n_seeds, P, l3, h3, perm, n_events, stream);
        case 8: return launch_sort_e<8>(seeds, n_seeds, P, l3, h3, perm, n_events, stream);
        case 16: return launch_sort_e<16>(seeds, n_seeds, P, l3, h3, perm, n_events, stream);
    }
    return cudaErrorInvalidValue;  // n_seeds > 16384 (multistart_culled_ok rejects it first)
}

template <int MODEL, int S, bool ZREF>
static cudaError_t launch_mc(const MultistartArgs &a0, int n_events, int32_t *perm, unsigned long long *pairs_evaluated,
                             cudaStream_t stream) {
    constexpr int P = (MODEL == kSlope3) ? 3 : 2;
    cudaError_t err = launch_seed_morton_sort(a0.seeds, a0.n_seeds, P, a0.lo, a0.hi, perm, n_events, stream);
    if (err != cudaSuccess) return err;
    MultistartArgs a = a0;
    a.cap = ((std::max(a0.cap, 2) + 7) / 8) * 8;  // resident stage (events beyond it run dense)
    const size_t smem = (size_t)a.cap * (sizeof(float4) + kMcWarps * sizeof(uint16_t));
    auto kern = multistart_culled_kernel<MODEL, S, ZREF>;
    err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    // units per block: up to kMcUnits, fewer when the launch would not give ~3 blocks per slot
    constexpr int useeds = 32 * S;
    const long long units_all = (long long)n_events * ((a.n_seeds + useeds - 1) / useeds);
    int upc = (int)std::min<long long>(kMcUnits, units_all / (3LL * 148 * RETINA_MC_MINB));
    upc = std::max(upc, kMcWarps);
    const int blocks = (a.n_seeds + upc * useeds - 1) / (upc * useeds);
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        const int ne = std::min(65535, n_events - e0);
        a.e_base = e0;
        kern<<<dim3(blocks, ne), kMcThreads, smem, stream>>>(a, perm, pairs_evaluated, upc);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

cudaError_t launch_multistart_culled(int model, const MultistartArgs &a, int n_events, int32_t *perm,
                                     unsigned long long *pairs_evaluated, cudaStream_t stream) {
    if (n_events == 0 || a.n_seeds == 0) return cudaSuccess;
    if (model == kSlope3) return launch_mc<kSlope3, RETINA_MC3_SEEDS, false>(a, n_events, perm, pairs_evaluated, stream);
    if (model != kSlope2) return cudaErrorInvalidValue;
    return (a.z_ref == 0.f) ? launch_mc<kSlope2, kMcSeeds, false>(a, n_events, perm, pairs_evaluated, stream)
                            : launch_mc<kSlope2, kMcSeeds, true>(a, n_events, perm, pairs_evaluated, stream);
}

}  // namespace retina
