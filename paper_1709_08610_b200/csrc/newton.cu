// newton.cu -- K6: the paper's own update (NEXT #1): Algorithm 1 with
// update[.] = one Truncated-Newton step per optimisation step j = 1..q at bandwidth sigma_j,
// using R, grad R and the Hessian H R computed in ONE pass over the hits.
//
// Per seed and step j (readings Z22-Z25, oracle.c ora_newton):
//   R0, g, H = eval(theta, sigma_j)                                   (1 pass, Hessian mode)
//   p = truncated CG on (-H) p = g, <= P iterations; non-positive curvature stops it, or at the
//       first iteration falls back to p = eta_j g
//   alpha = 1, 1/2, ... (<= max_halvings halvings): theta_t = clamp(theta + alpha p);
//       accept the first theta_t with R(theta_t) >= R0 + 1e-4 alpha g.p  (1 R-only pass each;
//       the CTA keeps passing while any of its seeds is still searching)
// then R (and grad R) at final_sigma.
//
// Hessian accumulation (SLOPE2 / SLOPE3; A = s_x, B = s_y, c = 2/sigma^2, d = z - z_ref or z - z0):
// per detector plane the loop sums W = sum w, wA, wB, wA^2, wAB, wB^2 (8 FMA-pipe ops per pair
// on top of the residual/exponent), and at each plane change folds them into accumulators
// weighted by 1, d and d^2, from which
//   g_tx = c sum d wA,  g_ty = c sum d wB,  g_z0 = -c (tx sum wA + ty sum wB)
//   H_txtx = c^2 sum d^2 wA^2 - c sum d^2 w,  H_tyty = c^2 sum d^2 wB^2 - c sum d^2 w,
//   H_txty = c^2 sum d^2 wAB,
//   H_txz0 = -c^2 (tx sum d wA^2 + ty sum d wAB) + c tx sum d w - c sum wA,
//   H_tyz0 = -c^2 (tx sum d wAB + ty sum d wB^2) + c ty sum d w - c sum wB,
//   H_z0z0 = c^2 (tx^2 sum wA^2 + 2 tx ty sum wAB + ty^2 sum wB^2) - c (tx^2 + ty^2) sum w.
//
// K6c (CULL, RETINA_MS_CULLED, SLOPE2): the same kernel, each warp visiting only the hits that can
// contribute (a skipped hit's ex2.approx.ftz weight is exactly +0, cull.cuh), one launch per Newton
// step with the seeds re-sorted by their current theta before each -- see newton_kernel.
#include "common.cuh"
#include "kernels.cuh"
#include "cull.cuh"

#include <algorithm>

namespace retina {

constexpr int kNtThreads = 128;

// Plane-weighted sums for one seed.  Index: [0] w [1] wA [2] wB [3] wA2 [4] wAB [5] wB2.
struct HessSums {
    float p[6];    // current plane
    float s1[6];   // weight 1 (s1[0] = R)
    float sd[6];   // weight d
    float sd2[6];  // weight d^2
};

// K6c: a pass restricted to the resident hits within reach of the box of the warp's points (cull.cuh):
// the hits are copied kNtChunk at a time into the warp's list buffer, each chunk's list consumed in
// hit order before the next is built (a copy, not an index: the pass then reads its hits in order,
// with no dependent shared-memory load per hit).
#ifndef RETINA_NT_CHUNK
#define RETINA_NT_CHUNK 128  // hits listed per chunk (the list buffer of a warp: 2 KB)
#endif
constexpr int kNtChunk = RETINA_NT_CHUNK;
struct NtReach {
    McBox box;
    float K;         // 1 / sigma^2 of the pass
    float4 *list;    // the warp's kNtChunk-entry buffer; nullptr: every hit (dense pass)
};

// Visits the event's hits in order: all of them (streamed or resident), or (rc.list != nullptr) only
// the resident hits within reach -- a skipped hit would add exactly +0.  Returns the hits visited.
template <int MODEL, bool ZREF, class F>
__device__ __forceinline__ int nt_visit(HitStage &st, const NtReach &rc, float zref, F &&f) {
    if (rc.list != nullptr) {
        const float4 *h = st.buf;
        int visited = 0;
        for (int k0 = 0; k0 < st.n; k0 += kNtChunk) {
            const int L = mc_build_list_range<MODEL, ZREF>(h, k0, min(st.n, k0 + kNtChunk), rc.box, rc.K, zref,
                                                           rc.list);
            RETINA_ASSERT(L >= 0 && L <= kNtChunk);
            visited += L;
#pragma unroll 2
            for (int t = 0; t < L; ++t) f(rc.list[t]);
            __syncwarp();  // the list is rebuilt next
        }
        return visited;
    } else {
        st.pass([&](const float4 *h, int len) {
#pragma unroll 2
            for (int k = 0; k < len; ++k) f(h[k]);
        });
        return st.n;
    }
}

template <int MODEL, int S, bool ZREF>
__device__ __forceinline__ int nt_pass_hess(HitStage &st, const float (&th)[S][3], float negK, float zref,
                                             HessSums (&hs)[S], const NtReach &rc = NtReach{{}, 0.f, nullptr}) {
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
        for (int q = 0; q < 6; ++q) hs[s].p[q] = hs[s].s1[q] = hs[s].sd[q] = hs[s].sd2[q] = 0.f;
    float dh[S], dl[S];
#pragma unroll
    for (int s = 0; s < S; ++s) dh[s] = dl[s] = 0.f;
    float zprev = __int_as_float(0x7fc00000);
    auto flush = [&]() {
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const float d = dh[s], d2 = __fmul_rn(dh[s], dh[s]);
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                hs[s].s1[q] = __fadd_rn(hs[s].s1[q], hs[s].p[q]);
                hs[s].sd[q] = __fmaf_rn(d, hs[s].p[q], hs[s].sd[q]);
                hs[s].sd2[q] = __fmaf_rn(d2, hs[s].p[q], hs[s].sd2[q]);
                hs[s].p[q] = 0.f;
            }
        }
    };
    const int visited = nt_visit<MODEL, ZREF>(st, rc, zref, [&](const float4 hk) {
        if (hk.z != zprev) {  // warp-uniform plane change
            flush();
            zprev = hk.z;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (MODEL == kSlope3)
                    two_sum(hk.z, -th[s][2], dh[s], dl[s]);
                else if (ZREF)
                    two_sum(hk.z, -zref, dh[s], dl[s]);
                else {
                    dh[s] = hk.z;
                    dl[s] = 0.f;
                }
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            float A, B;
            if (MODEL == kSlope3 || ZREF) {
                A = __fmaf_rn(-th[s][0], dl[s], __fmaf_rn(-th[s][0], dh[s], hk.x));
                B = __fmaf_rn(-th[s][1], dl[s], __fmaf_rn(-th[s][1], dh[s], hk.y));
            } else {
                A = __fmaf_rn(-th[s][0], hk.z, hk.x);
                B = __fmaf_rn(-th[s][1], hk.z, hk.y);
            }
            const float w = ex2_approx(__fmul_rn(__fmaf_rn(A, A, __fmul_rn(B, B)), negK));
            const float wA = __fmul_rn(w, A), wB = __fmul_rn(w, B);
            hs[s].p[0] = __fadd_rn(hs[s].p[0], w);
            hs[s].p[1] = __fadd_rn(hs[s].p[1], wA);
            hs[s].p[2] = __fadd_rn(hs[s].p[2], wB);
            hs[s].p[3] = __fmaf_rn(wA, A, hs[s].p[3]);
            hs[s].p[4] = __fmaf_rn(wA, B, hs[s].p[4]);
            hs[s].p[5] = __fmaf_rn(wB, B, hs[s].p[5]);
        }
    });
    flush();
    return visited;
}

// R only (line-search trials and the final pass); grad too when GRAD.
template <int MODEL, int S, bool ZREF, bool GRAD>
__device__ __forceinline__ int nt_pass_r(HitStage &st, const float (&th)[S][3], float negK, float zref,
                                          float (&R)[S], float (&G)[S][4], const NtReach &rc = NtReach{{}, 0.f, nullptr}) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
        R[s] = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) G[s][q] = 0.f;
    }
    float dh[S], dl[S], qa[S], qb[S];
#pragma unroll
    for (int s = 0; s < S; ++s) dh[s] = dl[s] = qa[s] = qb[s] = 0.f;
    float zprev = __int_as_float(0x7fc00000);
    auto flush = [&]() {
        if constexpr (GRAD) {
#pragma unroll
            for (int s = 0; s < S; ++s) {
                G[s][0] = __fmaf_rn(dh[s], qa[s], G[s][0]);
                G[s][1] = __fmaf_rn(dh[s], qb[s], G[s][1]);
                G[s][2] = __fadd_rn(G[s][2], qa[s]);
                G[s][3] = __fadd_rn(G[s][3], qb[s]);
                qa[s] = qb[s] = 0.f;
            }
        }
    };
    const int visited = nt_visit<MODEL, ZREF>(st, rc, zref, [&](const float4 hk) {
        if (hk.z != zprev) {
            flush();
            zprev = hk.z;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (MODEL == kSlope3)
                    two_sum(hk.z, -th[s][2], dh[s], dl[s]);
                else if (ZREF)
                    two_sum(hk.z, -zref, dh[s], dl[s]);
                else {
                    dh[s] = hk.z;
                    dl[s] = 0.f;
                }
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            float A, B;
            if (MODEL == kSlope3 || ZREF) {
                A = __fmaf_rn(-th[s][0], dl[s], __fmaf_rn(-th[s][0], dh[s], hk.x));
                B = __fmaf_rn(-th[s][1], dl[s], __fmaf_rn(-th[s][1], dh[s], hk.y));
            } else {
                A = __fmaf_rn(-th[s][0], hk.z, hk.x);
                B = __fmaf_rn(-th[s][1], hk.z, hk.y);
            }
            const float w = ex2_approx(__fmul_rn(__fmaf_rn(A, A, __fmul_rn(B, B)), negK));
            R[s] = __fadd_rn(R[s], w);
            if (GRAD) {
                qa[s] = __fmaf_rn(w, A, qa[s]);
                qb[s] = __fmaf_rn(w, B, qb[s]);
            }
        }
    });
    flush();
    return visited;
}

// Packed variants of the two passes above for seed PAIRS (FFMA2 / FMUL2 / FADD2): the same
// operation sequence per seed, each half an independent IEEE round-to-nearest operation, so
// the results are bit-identical to nt_pass_hess / nt_pass_r with half the issue slots.
template <int MODEL, int S, bool ZREF>
__device__ __forceinline__ int nt_pass_hess_x2(HitStage &st, const float (&th)[S][3], float negK, float zref,
                                                HessSums (&hs)[S], const NtReach &rc = NtReach{{}, 0.f, nullptr}) {
    static_assert(S % 2 == 0, "seed pairs");
    constexpr int NP = S / 2;
    const float2 zero = make_float2(0.f, 0.f), nk = make_float2(negK, negK);
    float2 mtx[NP], mty[NP], dh[NP], dl[NP], pp[NP][6], s1[NP][6], sd[NP][6], sd2[NP][6];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        mtx[p] = make_float2(-th[2 * p][0], -th[2 * p + 1][0]);
        mty[p] = make_float2(-th[2 * p][1], -th[2 * p + 1][1]);
        dh[p] = dl[p] = zero;
#pragma unroll
        for (int q = 0; q < 6; ++q) pp[p][q] = s1[p][q] = sd[p][q] = sd2[p][q] = zero;
    }
    float zprev = __int_as_float(0x7fc00000);
    auto flush = [&]() {
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const float2 d = dh[p], d2 = __fmul2_rn(dh[p], dh[p]);
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                s1[p][q] = __fadd2_rn(s1[p][q], pp[p][q]);
                sd[p][q] = __ffma2_rn(d, pp[p][q], sd[p][q]);
                sd2[p][q] = __ffma2_rn(d2, pp[p][q], sd2[p][q]);
                pp[p][q] = zero;
            }
        }
    };
    const int visited = nt_visit<MODEL, ZREF>(st, rc, zref, [&](const float4 hk) {
        if (hk.z != zprev) {  // warp-uniform plane change
            flush();
            zprev = hk.z;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                if (MODEL == kSlope3) {
                    two_sum(hk.z, -th[2 * p][2], dh[p].x, dl[p].x);
                    two_sum(hk.z, -th[2 * p + 1][2], dh[p].y, dl[p].y);
                } else if (ZREF) {
                    float hi, lo;
                    two_sum(hk.z, -zref, hi, lo);
                    dh[p] = make_float2(hi, hi);
                    dl[p] = make_float2(lo, lo);
                } else {
                    dh[p] = make_float2(hk.z, hk.z);
                }
            }
        }
        const float2 X = make_float2(hk.x, hk.x), Y = make_float2(hk.y, hk.y);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float2 A, B;
            if (MODEL == kSlope3 || ZREF) {
                A = __ffma2_rn(mtx[p], dl[p], __ffma2_rn(mtx[p], dh[p], X));
                B = __ffma2_rn(mty[p], dl[p], __ffma2_rn(mty[p], dh[p], Y));
            } else {
                const float2 Z = make_float2(hk.z, hk.z);
                A = __ffma2_rn(mtx[p], Z, X);
                B = __ffma2_rn(mty[p], Z, Y);
            }
            const float2 a = __fmul2_rn(__ffma2_rn(A, A, __fmul2_rn(B, B)), nk);
            const float2 w = make_float2(ex2_approx(a.x), ex2_approx(a.y));
            const float2 wA = __fmul2_rn(w, A), wB = __fmul2_rn(w, B);
            pp[p][0] = __fadd2_rn(pp[p][0], w);
            pp[p][1] = __fadd2_rn(pp[p][1], wA);
            pp[p][2] = __fadd2_rn(pp[p][2], wB);
            pp[p][3] = __ffma2_rn(wA, A, pp[p][3]);
            pp[p][4] = __ffma2_rn(wA, B, pp[p][4]);
            pp[p][5] = __ffma2_rn(wB, B, pp[p][5]);
        }
    });
    flush();
#pragma unroll
    for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            hs[2 * p].s1[q] = s1[p][q].x;
            hs[2 * p + 1].s1[q] = s1[p][q].y;
            hs[2 * p].sd[q] = sd[p][q].x;
            hs[2 * p + 1].sd[q] = sd[p][q].y;
            hs[2 * p].sd2[q] = sd2[p][q].x;
            hs[2 * p + 1].sd2[q] = sd2[p][q].y;
        }
    return visited;
}

template <int MODEL, int S, bool ZREF, bool GRAD>
__device__ __forceinline__ int nt_pass_r_x2(HitStage &st, const float (&th)[S][3], float negK, float zref,
                                             float (&R)[S], float (&G)[S][4], const NtReach &rc = NtReach{{}, 0.f, nullptr}) {
    static_assert(S % 2 == 0, "seed pairs");
    constexpr int NP = S / 2;
    const float2 zero = make_float2(0.f, 0.f), nk = make_float2(negK, negK);
    float2 mtx[NP], mty[NP], dh[NP], dl[NP], r2[NP], qa[NP], qb[NP], g[NP][4];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        mtx[p] = make_float2(-th[2 * p][0], -th[2 * p + 1][0]);
        mty[p] = make_float2(-th[2 * p][1], -th[2 * p + 1][1]);
        dh[p] = dl[p] = r2[p] = qa[p] = qb[p] = zero;
#pragma unroll
        for (int q = 0; q < 4; ++q) g[p][q] = zero;
    }
    float zprev = __int_as_float(0x7fc00000);
    auto flush = [&]() {
        if constexpr (GRAD) {
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                g[p][0] = __ffma2_rn(dh[p], qa[p], g[p][0]);
                g[p][1] = __ffma2_rn(dh[p], qb[p], g[p][1]);
                g[p][2] = __fadd2_rn(g[p][2], qa[p]);
                g[p][3] = __fadd2_rn(g[p][3], qb[p]);
                qa[p] = qb[p] = zero;
            }
        }
    };
    const int visited = nt_visit<MODEL, ZREF>(st, rc, zref, [&](const float4 hk) {
        if (hk.z != zprev) {
            flush();
            zprev = hk.z;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                if (MODEL == kSlope3) {
                    two_sum(hk.z, -th[2 * p][2], dh[p].x, dl[p].x);
                    two_sum(hk.z, -th[2 * p + 1][2], dh[p].y, dl[p].y);
                } else if (ZREF) {
                    float hi, lo;
                    two_sum(hk.z, -zref, hi, lo);
                    dh[p] = make_float2(hi, hi);
                    dl[p] = make_float2(lo, lo);
                } else {
                    dh[p] = make_float2(hk.z, hk.z);
                }
            }
        }
        const float2 X = make_float2(hk.x, hk.x), Y = make_float2(hk.y, hk.y);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            float2 A, B;
            if (MODEL == kSlope3 || ZREF) {
                A = __ffma2_rn(mtx[p], dl[p], __ffma2_rn(mtx[p], dh[p], X));
                B = __ffma2_rn(mty[p], dl[p], __ffma2_rn(mty[p], dh[p], Y));
            } else {
                const float2 Z = make_float2(hk.z, hk.z);
                A = __ffma2_rn(mtx[p], Z, X);
                B = __ffma2_rn(mty[p], Z, Y);
            }
            const float2 a = __fmul2_rn(__ffma2_rn(A, A, __fmul2_rn(B, B)), nk);
            const float2 w = make_float2(ex2_approx(a.x), ex2_approx(a.y));
            r2[p] = __fadd2_rn(r2[p], w);
            if (GRAD) {
                qa[p] = __ffma2_rn(w, A, qa[p]);
                qb[p] = __ffma2_rn(w, B, qb[p]);
            }
        }
    });
    flush();
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        R[2 * p] = r2[p].x;
        R[2 * p + 1] = r2[p].y;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            G[2 * p][q] = g[p][q].x;
            G[2 * p + 1][q] = g[p][q].y;
        }
    }
    return visited;
}

#ifndef RETINA_NT_MINB
#define RETINA_NT_MINB 4  // CTAs per SM the register allocation must allow (5: 96 registers + spills, 2 % slower)
#endif
#ifndef RETINA_NT3_MINB
#define RETINA_NT3_MINB 3  // SLOPE3 (4 seeds x 3 parameters per thread: 154 registers, no spills)
#endif
#ifndef RETINA_NTC_SEEDS
#define RETINA_NTC_SEEDS 2  // K6c (SLOPE2) seeds per thread (64-seed warps: tighter boxes, 17 % of the pairs instead of 23 %; cfg3 9.63 -> 9.34 ms per 1,000 events)
#endif
#ifndef RETINA_NTC_MINB
#define RETINA_NTC_MINB 5  // K6c CTAs per SM the register allocation must allow (6 / 7: 9.90 / 9.80 ms)
#endif
#ifndef RETINA_NT_X2
#define RETINA_NT_X2 1  // packed seed-pair passes (0: scalar reference passes)
#endif

// Truncated CG on (-H) p = g (maximisation), <= P iterations, fallback eta g (oracle tn_direction).
// The solve runs in fp64 on the fp32-accumulated g and H: for SLOPE3 the Hessian's scales differ by
// ~(d / t)^2 ~ 1e7 between the slope and z0 axes, so an fp32 CG loses the z0 component of the
// Newton direction (round 2: 7.6 % of cfg4 seeds ended > 1e-3 x range from the oracle); in fp64 the
// only error left is the elementwise-relative accumulation error of g and H, which the scaling does
// not amplify.  P <= 3: a few dozen DFMA per seed per Newton step, nothing next to its hit passes.
template <int P>
__device__ __forceinline__ void nt_direction(const float (&g)[3], const float (&H)[3][3], float eta, float (&p)[3]) {
    double x[3] = {0.0, 0.0, 0.0}, r[3], d[3], Ad[3];
    double rr = 0.0;
#pragma unroll
    for (int a = 0; a < P; ++a) {
        r[a] = g[a];
        d[a] = g[a];
        rr = fma((double)g[a], (double)g[a], rr);
    }
    const double rr0 = rr;
#pragma unroll
    for (int it = 0; it < P; ++it) {
        if (!(rr > 0.0)) break;
        double curv = 0.0;
#pragma unroll
        for (int a = 0; a < P; ++a) {
            double v = 0.0;
#pragma unroll
            for (int b = 0; b < P; ++b) v = fma(-(double)H[a][b], d[b], v);
            Ad[a] = v;
            curv = fma(d[a], v, curv);
        }
        if (!(curv > 0.0)) {
            if (it == 0) {
#pragma unroll
                for (int a = 0; a < P; ++a) x[a] = (double)eta * (double)g[a];
            }
            break;
        }
        const double alpha = rr / curv;
        double rr_new = 0.0;
#pragma unroll
        for (int a = 0; a < P; ++a) {
            x[a] = fma(alpha, d[a], x[a]);
            r[a] = fma(-alpha, Ad[a], r[a]);
            rr_new = fma(r[a], r[a], rr_new);
        }
        if (rr_new <= 1e-24 * rr0) break;
        const double beta = rr_new / rr;
#pragma unroll
        for (int a = 0; a < P; ++a) d[a] = fma(beta, d[a], r[a]);
        rr = rr_new;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a) p[a] = (a < P) ? (float)x[a] : 0.f;
}

// Shared state of the compacted line search: per seed slot (owner thread t, seed s -> slot
// s * kNtThreads + t) the base point, direction, R0 and Armijo slope, and two queues of slots.
template <int S, int P>
struct LineSearchSmem {
    float base[kNtThreads * S][P];  // theta before the step; the accepted trial overwrites it
    float dir[kNtThreads * S][P];
    float R0[kNtThreads * S], slope[kNtThreads * S];
    // (k << 32) | bits(R_t) of the smallest halving k of the current round that passed Armijo:
    // one 64-bit atomicMin keeps both the decision and that trial's response
    // (all ones: no halving accepted yet); also gives the halvings tried and the final response
    unsigned long long kmin[kNtThreads * S];
    int q[2][kNtThreads * S];
    int nq[2];
};

// Halvings k = 1 .. max_halvings for the seeds still active after the alpha = 1 trial.
// Worker thread (warp w, lane l) takes queue entries w * 32 SQ + s * 32 + l, s < SQ; warps past
// the queue's end skip the pass.  Needs the hits resident (pass() then has no barrier).
#ifndef RETINA_NT_SQ
#define RETINA_NT_SQ 1  // queue entries per worker thread (1 measured best: C0 5.3 vs 6.0 (2), 7.8 (4) on cfg3)
#endif
#ifndef RETINA_NT3_SQ
#define RETINA_NT3_SQ 2  // SLOPE3: two entries per worker as one packed seed pair (cfg4 Newton 15.55 -> 15.08 ms per 100 events)
#endif
#ifndef RETINA_NT_LSB
#define RETINA_NT_LSB 4  // halvings evaluated together per queue round (measured: C0 4.9 / 4.0 / 3.8 / 3.8 for 1 / 2 / 4 / 8)
#endif
constexpr int kNtLsBatch = RETINA_NT_LSB;
template <int MODEL, int S, bool ZREF, bool CULL>
__device__ __forceinline__ void nt_line_search_queue(HitStage &st, const NewtonArgs &a, float negK, float (&th)[S][3],
                                                     const float (&p)[S][3], const float (&R0)[S],
                                                     const float (&slope)[S], const bool (&active)[S], int (&nev)[S],
                                                     float (&rcur)[S], LineSearchSmem<S, (MODEL == kSlope3) ? 3 : 2> &ls,
                                                     float4 *list, unsigned long long &evaluated) {
    constexpr int P = (MODEL == kSlope3) ? 3 : 2;
    constexpr int SQW = (MODEL == kSlope3) ? RETINA_NT3_SQ : RETINA_NT_SQ;
    constexpr int SQ = SQW < S ? SQW : S;
    const int tid = threadIdx.x, lane = tid & 31, wbase = (tid >> 5) * 32 * SQ;
    __syncthreads();  // previous users of ls are done
    if (tid == 0) ls.nq[0] = ls.nq[1] = 0;
    __syncthreads();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (!active[s]) continue;
        const int slot = s * kNtThreads + tid;
#pragma unroll
        for (int i = 0; i < P; ++i) {
            ls.base[slot][i] = th[s][i];
            ls.dir[slot][i] = p[s][i];
        }
        ls.R0[slot] = R0[s];
        ls.slope[slot] = slope[s];
        ls.kmin[slot] = ~0ull;
        ls.q[0][atomicAdd(&ls.nq[0], 1)] = slot;
    }
    __syncthreads();
    // Rounds of LB halvings: every (queued seed, k) pair of the round is one entry, all evaluated
    // in the same pass; the seed takes the smallest k whose trial passes Armijo (exactly the
    // sequential rule's choice -- the later trials of the round are speculative work).
    int cur = 0;
    for (int k0 = 1; k0 <= a.max_halvings; k0 += kNtLsBatch) {
        const int nb = min(kNtLsBatch, a.max_halvings - k0 + 1);
        const int n = ls.nq[cur];  // final: written before the last barrier
        if (n == 0) break;
        const int ne = n * nb;
        for (int wb = wbase; wb < ne; wb += kNtThreads * SQ) {  // ne may exceed one sweep of the CTA
            int slot[SQ], kk[SQ];
            float tt[SQ][3];
#pragma unroll
            for (int s = 0; s < SQ; ++s) {
                const int e = wb + s * 32 + lane;
                const bool valid = e < ne;
                const int qi = valid ? e / nb : 0;  // padding lanes repeat entry 0
                kk[s] = k0 + (valid ? e - qi * nb : 0);
                const int src = ls.q[cur][qi];
                slot[s] = valid ? src : -1;
                const float alpha = __int_as_float((127 - kk[s]) << 23);  // 2^-k, exact
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    tt[s][i] = (i < P) ? fminf(fmaxf(__fmaf_rn(alpha, ls.dir[src][i], ls.base[src][i]), a.lo[i]),
                                               a.hi[i])
                                       : 0.f;
            }
            // K6c (list != nullptr): the hits within reach of this worker warp's trial points
            NtReach rq{{}, 0.f, nullptr};
            int nv = 0;
            if constexpr (CULL) {
                bool okq[SQ];
#pragma unroll
                for (int s = 0; s < SQ; ++s) {
                    okq[s] = slot[s] >= 0;
                    nv += okq[s] ? 1 : 0;
                }
                nv = __reduce_add_sync(0xffffffffu, nv);
                rq = NtReach{mc_warp_box<P, SQ>(tt, okq), -negK, list};
            }
            float Rt[SQ], Gd[SQ][4];
            int vis;
            if constexpr (RETINA_NT_X2 && SQ % 2 == 0)
                vis = nt_pass_r_x2<MODEL, SQ, ZREF, false>(st, tt, negK, a.z_ref, Rt, Gd, rq);
            else
                vis = nt_pass_r<MODEL, SQ, ZREF, false>(st, tt, negK, a.z_ref, Rt, Gd, rq);
            if constexpr (CULL) evaluated += (unsigned long long)vis * nv;
#pragma unroll
            for (int s = 0; s < SQ; ++s) {
                if (slot[s] < 0) continue;
                const int sl = slot[s];
                const float alpha = __int_as_float((127 - kk[s]) << 23);
                if (Rt[s] >= __fmaf_rn(1e-4f * alpha, ls.slope[sl], ls.R0[sl]))
                    atomicMin(&ls.kmin[sl], ((unsigned long long)kk[s] << 32) | __float_as_uint(Rt[s]));
            }
        }
        __syncthreads();  // every trial of the round is decided
        for (int i = tid; i < n; i += kNtThreads) {
            const int sl = ls.q[cur][i];
            const unsigned long long kr = ls.kmin[sl];
            const int km = (kr == ~0ull) ? 0x7fffffff : (int)(kr >> 32);
            if (km < k0 + nb) {  // accepted: recompute the trial point (same operations, same bits)
                const float alpha = __int_as_float((127 - km) << 23);
#pragma unroll
                for (int d = 0; d < P; ++d)
                    ls.base[sl][d] = fminf(fmaxf(__fmaf_rn(alpha, ls.dir[sl][d], ls.base[sl][d]), a.lo[d]), a.hi[d]);
            } else {
                ls.q[cur ^ 1][atomicAdd(&ls.nq[cur ^ 1], 1)] = sl;
            }
        }
        __syncthreads();  // all reads of queue cur and all pushes to cur ^ 1 are done
        if (tid == 0) ls.nq[cur] = 0;
        cur ^= 1;
        __syncthreads();
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (!active[s]) continue;
        const int slot = s * kNtThreads + tid;
#pragma unroll
        for (int i = 0; i < P; ++i) th[s][i] = ls.base[slot][i];
        const unsigned long long kr = ls.kmin[slot];
        if (kr == ~0ull) {
            nev[s] += a.max_halvings;  // every halving tried, none accepted: theta and R(theta) stay
        } else {
            nev[s] += (int)(kr >> 32);
            rcur[s] = __uint_as_float((uint32_t)kr);  // response at the accepted trial point
        }
    }
}

// The same halvings with a queue per WARP: the warp's own seeds still searching after the alpha = 1
// trial are compacted (ballot) into its own part of ls.q, and the warp alone evaluates their
// (seed, k) entries, 32 SQ per pass: no block barrier, so warps whose passes differ in length (K6c's
// lists) never wait for each other, and (K6c) a pass's trial points all come from the warp's
// Morton-neighbouring seeds.  Same entries, same decisions, same bits as the block-wide queue.
template <int MODEL, int S, bool ZREF, bool CULL>
__device__ __forceinline__ void nt_line_search_warp(HitStage &st, const NewtonArgs &a, float negK, float (&th)[S][3],
                                                    const float (&p)[S][3], const float (&R0)[S],
                                                    const float (&slope)[S], const bool (&active)[S], int (&nev)[S],
                                                    float (&rcur)[S], LineSearchSmem<S, (MODEL == kSlope3) ? 3 : 2> &ls,
                                                    float4 *list, unsigned long long &evaluated) {
    constexpr int P = (MODEL == kSlope3) ? 3 : 2;
    constexpr int SQW = (MODEL == kSlope3) ? RETINA_NT3_SQ : RETINA_NT_SQ;
    constexpr int SQ = SQW < S ? SQW : S;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned lt = (1u << lane) - 1u;
    int *qa = ls.q[0] + warp * 32 * S, *qb = ls.q[1] + warp * 32 * S;  // this warp's two queues
    __syncwarp();  // the warp's previous reads of ls are done
    int n = 0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
        const int slot = s * kNtThreads + tid;
        if (active[s]) {
#pragma unroll
            for (int i = 0; i < P; ++i) {
                ls.base[slot][i] = th[s][i];
                ls.dir[slot][i] = p[s][i];
            }
            ls.R0[slot] = R0[s];
            ls.slope[slot] = slope[s];
            ls.kmin[slot] = ~0ull;
        }
        const unsigned b = __ballot_sync(0xffffffffu, active[s]);
        if (active[s]) qa[n + __popc(b & lt)] = slot;
        n += __popc(b);
    }
    RETINA_ASSERT(n <= 32 * S);
    __syncwarp();
    for (int k0 = 1; k0 <= a.max_halvings && n > 0; k0 += kNtLsBatch) {
        const int nb = min(kNtLsBatch, a.max_halvings - k0 + 1);
        const int ne = n * nb;
        for (int wb = 0; wb < ne; wb += 32 * SQ) {
            int slot[SQ], kk[SQ];
            float tt[SQ][3];
#pragma unroll
            for (int s = 0; s < SQ; ++s) {
                const int e = wb + s * 32 + lane;
                const bool valid = e < ne;
                const int qi = valid ? e / nb : 0;  // padding lanes repeat entry 0
                kk[s] = k0 + (valid ? e - qi * nb : 0);
                const int src = qa[qi];
                slot[s] = valid ? src : -1;
                const float alpha = __int_as_float((127 - kk[s]) << 23);  // 2^-k, exact
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    tt[s][i] = (i < P) ? fminf(fmaxf(__fmaf_rn(alpha, ls.dir[src][i], ls.base[src][i]), a.lo[i]),
                                               a.hi[i])
                                       : 0.f;
            }
            NtReach rq{{}, 0.f, nullptr};
            int nv = 0;
            if constexpr (CULL) {
                bool okq[SQ];
#pragma unroll
                for (int s = 0; s < SQ; ++s) {
                    okq[s] = slot[s] >= 0;
                    nv += okq[s] ? 1 : 0;
                }
                nv = __reduce_add_sync(0xffffffffu, nv);
                rq = NtReach{mc_warp_box<P, SQ>(tt, okq), -negK, list};
            }
            float Rt[SQ], Gd[SQ][4];
            int vis;
            if constexpr (RETINA_NT_X2 && SQ % 2 == 0)
                vis = nt_pass_r_x2<MODEL, SQ, ZREF, false>(st, tt, negK, a.z_ref, Rt, Gd, rq);
            else
                vis = nt_pass_r<MODEL, SQ, ZREF, false>(st, tt, negK, a.z_ref, Rt, Gd, rq);
            if constexpr (CULL) evaluated += (unsigned long long)vis * nv;
#pragma unroll
            for (int s = 0; s < SQ; ++s) {
                if (slot[s] < 0) continue;
                const int sl = slot[s];
                const float alpha = __int_as_float((127 - kk[s]) << 23);
                if (Rt[s] >= __fmaf_rn(1e-4f * alpha, ls.slope[sl], ls.R0[sl]))
                    atomicMin(&ls.kmin[sl], ((unsigned long long)kk[s] << 32) | __float_as_uint(Rt[s]));
            }
        }
        __syncwarp();  // every trial of the round is decided
        int n2 = 0;
        for (int i0 = 0; i0 < n; i0 += 32) {
            const int i = i0 + lane;
            bool again = false;
            int sl = 0;
            if (i < n) {
                sl = qa[i];
                const unsigned long long kr = ls.kmin[sl];
                const int km = (kr == ~0ull) ? 0x7fffffff : (int)(kr >> 32);
                if (km < k0 + nb) {  // accepted: recompute the trial point (same operations, same bits)
                    const float alpha = __int_as_float((127 - km) << 23);
#pragma unroll
                    for (int d = 0; d < P; ++d)
                        ls.base[sl][d] =
                            fminf(fmaxf(__fmaf_rn(alpha, ls.dir[sl][d], ls.base[sl][d]), a.lo[d]), a.hi[d]);
                } else {
                    again = true;
                }
            }
            const unsigned b = __ballot_sync(0xffffffffu, again);
            if (again) qb[n2 + __popc(b & lt)] = sl;
            n2 += __popc(b);
        }
        __syncwarp();
        int *t = qa;
        qa = qb;
        qb = t;
        n = n2;
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (!active[s]) continue;
        const int slot = s * kNtThreads + tid;
#pragma unroll
        for (int i = 0; i < P; ++i) th[s][i] = ls.base[slot][i];
        const unsigned long long kr = ls.kmin[slot];
        if (kr == ~0ull) {
            nev[s] += a.max_halvings;  // every halving tried, none accepted: theta and R(theta) stay
        } else {
            nev[s] += (int)(kr >> 32);
            rcur[s] = __uint_as_float((uint32_t)kr);  // response at the accepted trial point
        }
    }
}

#ifndef RETINA_NT_WARPQ
#define RETINA_NT_WARPQ 2  // line-search queue per warp: bit 0 for K6, bit 1 for K6c (else block-wide; K6: cfg4 15.0 vs 16.2 ms per 100 events)
#endif

// CULL (K6c, RETINA_MS_CULLED): the same per-seed arithmetic and decisions, bit for bit, with each
// warp visiting only the hits within reach of its points (cull.cuh): the seeds are taken in the
// per-event Morton order perm (a warp holds 32 S consecutive ones, so its points stay in a small
// box), and the passes -- Hessian mode, the alpha = 1 trial, each line-search worker pass, the
// final pass -- list, chunk by chunk and in hit order, the resident hits that a conservative bound
// keeps within K s^2 <= 128 of the box of the points they evaluate.  K6c runs one launch per
// Newton step [a.j_begin, a.j_end) with the permutation re-sorted by the seeds' CURRENT theta
// before each (Newton steps move seeds far; re-sorting keeps every warp's points together), theta
// and the evaluation count carried in theta_out and the workspace between launches (a.first:
// theta from seeds; a.last: the final pass and every output).  Events larger than the stage run
// dense.  pairs_evaluated: CULL adds the pairs visited for real seeds; the dense kernel adds
// evaluations x hits.
template <int MODEL, int S, bool ZREF, bool CULL>
__global__ void __launch_bounds__(kNtThreads, CULL ? RETINA_NTC_MINB : (MODEL == kSlope3) ? RETINA_NT3_MINB : RETINA_NT_MINB)
    newton_kernel(NewtonArgs a, const int32_t *perm, unsigned long long *pairs_evaluated) {
    extern __shared__ __align__(16) float4 s_hits[];  // [cap] hits (K6c: then [warps][kNtChunk] listed hits)
    __shared__ __align__(8) uint64_t s_bar[2];
    constexpr int P = (MODEL == kSlope3) ? 3 : 2;

    const int e = a.e_base + blockIdx.y;
    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    HitStage st;
    st.init(s_hits, s_bar, a.hits + start, nh, a.cap);
    float4 *list = nullptr;  // this warp's list (K6c, resident events)
    if constexpr (CULL) {
        if (nh <= a.cap && nh <= 65535 && (nh == 0 || st.load_resident()))
            list = s_hits + a.cap + warp * kNtChunk;
    }
    unsigned long long evaluated = 0;  // (seed, hit) pairs this warp's passes evaluate for real seeds
    // a pass over the points pts (valid where ok): restricted to the hits in reach (K6c), or all of
    // them (nullptr); account() then adds its pairs
    int rc_nv = 0;
    auto reach = [&](const float (&pts)[S][3], const bool (&ok)[S], float K) {
        NtReach r{{}, 0.f, nullptr};
        if constexpr (CULL) {
            int nv = 0;
#pragma unroll
            for (int s = 0; s < S; ++s) nv += ok[s] ? 1 : 0;
            rc_nv = __reduce_add_sync(0xffffffffu, nv);
            r = NtReach{mc_warp_box<P, S>(pts, ok), K, list};
        }
        return r;
    };
    auto account = [&](int visited) {
        if constexpr (CULL) evaluated += (unsigned long long)visited * rc_nv;
    };

    int sid[S];  // position in the CTA's seed range (K6c: in the Morton order)
    bool valid[S];
    float th[S][3];
    // the caller's index of seed s
    auto orig = [&](int s) {
        if constexpr (CULL) {
            const int q = __ldg(perm + (int64_t)e * a.n_seeds + min(sid[s], a.n_seeds - 1));
            RETINA_ASSERT(q >= 0 && q < a.n_seeds);
            return q;
        } else {
            return min(sid[s], a.n_seeds - 1);
        }
    };
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if constexpr (CULL)
            sid[s] = blockIdx.x * (kNtThreads * S) + warp * (32 * S) + s * 32 + lane;
        else
            sid[s] = blockIdx.x * (kNtThreads * S) + s * kNtThreads + threadIdx.x;
        valid[s] = sid[s] < a.n_seeds;
        const int64_t src = ((int64_t)e * a.n_seeds + orig(s)) * P;
        const float *from = a.first ? a.seeds : a.theta_out;  // (written only by this thread, below)
#pragma unroll
        for (int i = 0; i < 3; ++i) th[s][i] = (i < P) ? from[src + i] : 0.f;
    }

    __shared__ LineSearchSmem<S, P> ls;
    HessSums hs[S];
    float R[S], G[S][4];
    int nev[S];     // response evaluations per seed (PAPER.md:200-201 cost unit)
    float Rcur[S];  // R(theta) at the current step's sigma: the last evaluation at the current point
#pragma unroll
    for (int s = 0; s < S; ++s) {
        // q Hessian-mode passes (+ the final one), or the count carried from the previous launch
        nev[s] = a.first ? a.n_steps + (a.reuse_final ? 0 : 1) : a.nev_ws[(int64_t)e * a.n_seeds + orig(s)];
        Rcur[s] = 0.f;
    }
    for (int j = a.j_begin; j < a.j_end; ++j) {
        const float c = a.c2[j], negK = a.negK[j];
        {
            const NtReach r = reach(th, valid, -negK);
            int vis;
            if constexpr (RETINA_NT_X2 && S % 2 == 0)
                vis = nt_pass_hess_x2<MODEL, S, ZREF>(st, th, negK, a.z_ref, hs, r);
            else
                vis = nt_pass_hess<MODEL, S, ZREF>(st, th, negK, a.z_ref, hs, r);
            account(vis);
        }
        float R0[S], p[S][3], slope[S], tt[S][3];
        bool active[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const float tx = th[s][0], ty = th[s][1];
            const float c2 = __fmul_rn(c, c);
            float g[3], H[3][3];
            R0[s] = hs[s].s1[0];
            Rcur[s] = R0[s];
            const float *s1 = hs[s].s1, *sd = hs[s].sd, *sd2 = hs[s].sd2;
            g[0] = __fmul_rn(c, sd[1]);
            g[1] = __fmul_rn(c, sd[2]);
            H[0][0] = __fmaf_rn(c2, sd2[3], -__fmul_rn(c, sd2[0]));
            H[1][1] = __fmaf_rn(c2, sd2[5], -__fmul_rn(c, sd2[0]));
            H[0][1] = H[1][0] = __fmul_rn(c2, sd2[4]);
            if (MODEL == kSlope3) {
                g[2] = -__fmul_rn(c, __fmaf_rn(tx, s1[1], __fmul_rn(ty, s1[2])));
                H[0][2] = H[2][0] = __fmaf_rn(-c2, __fmaf_rn(tx, sd[3], __fmul_rn(ty, sd[4])),
                                              __fmul_rn(c, __fmaf_rn(tx, sd[0], -s1[1])));
                H[1][2] = H[2][1] = __fmaf_rn(-c2, __fmaf_rn(tx, sd[4], __fmul_rn(ty, sd[5])),
                                              __fmul_rn(c, __fmaf_rn(ty, sd[0], -s1[2])));
                const float q = __fmaf_rn(tx * tx, s1[3], __fmaf_rn(2.f * tx * ty, s1[4], __fmul_rn(ty * ty, s1[5])));
                H[2][2] = __fmaf_rn(c2, q, -__fmul_rn(c, __fmul_rn(__fmaf_rn(tx, tx, ty * ty), s1[0])));
            } else {
                g[2] = 0.f;
                H[0][2] = H[2][0] = H[1][2] = H[2][1] = H[2][2] = 0.f;
            }
            nt_direction<P>(g, H, a.eta[j], p[s]);
            slope[s] = 0.f;
#pragma unroll
            for (int i = 0; i < P; ++i) slope[s] = __fmaf_rn(g[i], p[s][i], slope[s]);
            active[s] = valid[s];
        }
        // Trial alpha = 1 for every seed of the CTA (all owners pass over the hits together).
        // With the hits resident in shared memory, the seeds still searching after it are
        // compacted into a queue and later trials run only on the warps that hold queue
        // entries, so a halving costs ~ceil(active / (32 S)) warp passes instead of a whole CTA
        // pass (the oracle's per-seed loop, evaluated in a different thread: bit-identical).
        // Streaming events (hits > smem stage) keep the CTA-wide loop for every trial.
        const int kmax_cta = st.resident ? 0 : a.max_halvings;
        float alpha = 1.f;
        for (int k = 0; k <= kmax_cta; ++k, alpha *= 0.5f) {
            bool any = false;
#pragma unroll
            for (int s = 0; s < S; ++s) any |= active[s];
            // (resident hits: no barrier -- each warp's passes are its own; streamed: block-wide)
            if (st.resident ? !__any_sync(0xffffffffu, any) : !__syncthreads_or(any)) break;
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int i = 0; i < 3; ++i)
                    tt[s][i] = (i < P) ? fminf(fmaxf(__fmaf_rn(alpha, p[s][i], th[s][i]), a.lo[i]), a.hi[i]) : 0.f;
#pragma unroll
            for (int s = 0; s < S; ++s) nev[s] += active[s] ? 1 : 0;
            float Rt[S], Gd[S][4];
            const NtReach r = reach(tt, active, -negK);
            int vis;
            if constexpr (RETINA_NT_X2 && S % 2 == 0)
                vis = nt_pass_r_x2<MODEL, S, ZREF, false>(st, tt, negK, a.z_ref, Rt, Gd, r);
            else
                vis = nt_pass_r<MODEL, S, ZREF, false>(st, tt, negK, a.z_ref, Rt, Gd, r);
            account(vis);
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (active[s] && Rt[s] >= __fmaf_rn(1e-4f * alpha, slope[s], R0[s])) {
                    Rcur[s] = Rt[s];
#pragma unroll
                    for (int i = 0; i < 3; ++i) th[s][i] = tt[s][i];
                    active[s] = false;
                }
            }
        }
        if (st.resident && a.max_halvings > 0) {
            if constexpr ((RETINA_NT_WARPQ >> (CULL ? 1 : 0)) & 1)
                nt_line_search_warp<MODEL, S, ZREF, CULL>(st, a, negK, th, p, R0, slope, active, nev, Rcur, ls, list,
                                                          evaluated);
            else
                nt_line_search_queue<MODEL, S, ZREF, CULL>(st, a, negK, th, p, R0, slope, active, nev, Rcur, ls, list,
                                                           evaluated);
        }
    }
    if (!a.last) {  // K6c, a step launch before the last: carry theta and the evaluation count
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (valid[s]) {
                const int64_t o = (int64_t)e * a.n_seeds + orig(s);
                a.nev_ws[o] = nev[s];
#pragma unroll
                for (int i = 0; i < P; ++i) a.theta_out[o * P + i] = th[s][i];
            }
        }
        if (pairs_evaluated && lane == 0 && evaluated) atomicAdd(pairs_evaluated, evaluated);
        return;
    }
    float g[S][3];
    if (a.grad_out) {
        const NtReach r = reach(th, valid, -a.final_negK);
        int vis;
        if constexpr (RETINA_NT_X2 && S % 2 == 0)
            vis = nt_pass_r_x2<MODEL, S, ZREF, true>(st, th, a.final_negK, a.z_ref, R, G, r);
        else
            vis = nt_pass_r<MODEL, S, ZREF, true>(st, th, a.final_negK, a.z_ref, R, G, r);
        account(vis);
#pragma unroll
        for (int s = 0; s < S; ++s) {
            g[s][0] = __fmul_rn(a.final_c2, G[s][0]);
            g[s][1] = __fmul_rn(a.final_c2, G[s][1]);
            g[s][2] = (MODEL == kSlope3)
                          ? -__fmul_rn(a.final_c2, __fmaf_rn(th[s][0], G[s][2], __fmul_rn(th[s][1], G[s][3])))
                          : 0.f;
        }
    } else if (a.reuse_final) {
        // final sigma == last step's sigma and no gradient wanted: R(theta^q) is the response of
        // the last step's accepted trial (same point, same sigma, same arithmetic as a final
        // pass) or, with no trial accepted, the last Hessian pass's R at the unchanged theta
#pragma unroll
        for (int s = 0; s < S; ++s) R[s] = Rcur[s];
    } else {
        const NtReach r = reach(th, valid, -a.final_negK);
        int vis;
        if constexpr (RETINA_NT_X2 && S % 2 == 0)
            vis = nt_pass_r_x2<MODEL, S, ZREF, false>(st, th, a.final_negK, a.z_ref, R, G, r);
        else
            vis = nt_pass_r<MODEL, S, ZREF, false>(st, th, a.final_negK, a.z_ref, R, G, r);
        account(vis);
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
        if (valid[s]) {
            const int64_t o = (int64_t)e * a.n_seeds + orig(s);
            a.R_out[o] = R[s];
            if (a.evals_out) a.evals_out[o] = nev[s];
#pragma unroll
            for (int i = 0; i < P; ++i) {
                a.theta_out[o * P + i] = th[s][i];
                if (a.grad_out) a.grad_out[o * P + i] = g[s][i];
            }
        }
    }
    if constexpr (!CULL) {  // every evaluation visits every hit: evaluations x hits
        int ne = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) ne += valid[s] ? nev[s] : 0;
        evaluated = (unsigned long long)__reduce_add_sync(0xffffffffu, ne) * nh;
    }
    if (pairs_evaluated && lane == 0 && evaluated) atomicAdd(pairs_evaluated, evaluated);
}

#ifndef RETINA_NT3_SEEDS
#define RETINA_NT3_SEEDS 4  // SLOPE3 seeds per thread (2 with 5 CTAs/SM: cfg4 Newton 33.5 vs 30.2 ms per 200 events)
#endif
template <int MODEL, bool ZREF, bool CULL>
static cudaError_t launch_nt(const NewtonArgs &a0, int n_events, const int32_t *perm,
                             unsigned long long *pairs_evaluated, cudaStream_t stream) {
    constexpr int S = CULL ? RETINA_NTC_SEEDS : (MODEL == kSlope3) ? RETINA_NT3_SEEDS : 4;
    auto kern = newton_kernel<MODEL, S, ZREF, CULL>;
    NewtonArgs a = a0;
    const size_t smem = (size_t)a.cap * sizeof(float4) + (CULL ? (kNtThreads / 32) * kNtChunk * sizeof(float4) : 0);
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const int blocks = (a.n_seeds + kNtThreads * S - 1) / (kNtThreads * S);
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        kern<<<dim3(blocks, ne), kNtThreads, smem, stream>>>(a, perm, pairs_evaluated);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

cudaError_t launch_newton(int model, const NewtonArgs &a0, int n_events, unsigned long long *pairs_evaluated,
                          cudaStream_t stream) {
    if (n_events == 0 || a0.n_seeds == 0) return cudaSuccess;
    NewtonArgs a = a0;  // every step in one launch
    a.j_begin = 0;
    a.j_end = a.n_steps;
    a.first = a.last = 1;
    switch (model) {
        case kSlope2:
            return (a.z_ref == 0.f) ? launch_nt<kSlope2, false, false>(a, n_events, nullptr, pairs_evaluated, stream)
                                    : launch_nt<kSlope2, true, false>(a, n_events, nullptr, pairs_evaluated, stream);
        case kSlope3: return launch_nt<kSlope3, false, false>(a, n_events, nullptr, pairs_evaluated, stream);
    }
    return cudaErrorInvalidValue;
}

size_t newton_culled_workspace_bytes(long long n_events, int n_seeds) {
    return (size_t)(n_events * n_seeds) * 2 * sizeof(int32_t);  // perm, then the evaluation counts
}

// SLOPE3 runs K6 (the dense kernel) under RETINA_MS_CULLED: its wide early sigma_j (x 6, x 3.5 of
// sigma = 0.88 mm on cfg4) and a warp box's z0 extent keep 80-97 % of the hits in reach
// (tools/k6c_reach.py), so listing costs more than it saves (cfg4, 100 events: 15.0 ms dense, 16.2
// culled).  The results are the same either way.
cudaError_t launch_newton_culled(int model, const NewtonArgs &a0, int n_events, int32_t *ws,
                                 unsigned long long *pairs_evaluated, cudaStream_t stream) {
    if (n_events == 0 || a0.n_seeds == 0) return cudaSuccess;
    if (model == kSlope3) return launch_newton(model, a0, n_events, pairs_evaluated, stream);
    if (model != kSlope2) return cudaErrorInvalidValue;
    constexpr int P = 2;
    int32_t *perm = ws;
    NewtonArgs a = a0;
    a.nev_ws = ws + (int64_t)n_events * a.n_seeds;
    const int launches = a.n_steps > 0 ? a.n_steps : 1;
    for (int j = 0; j < launches; ++j) {  // one Newton step per launch, the seeds re-sorted by theta first
        a.j_begin = j;
        a.j_end = a.n_steps > 0 ? j + 1 : 0;
        a.first = (j == 0);
        a.last = (j == launches - 1);
        cudaError_t err = launch_seed_morton_sort(j == 0 ? a.seeds : a.theta_out, a.n_seeds, P, a.lo, a.hi, perm,
                                                  n_events, stream);
        if (err != cudaSuccess) return err;
        err = (a.z_ref == 0.f) ? launch_nt<kSlope2, false, true>(a, n_events, perm, pairs_evaluated, stream)
                               : launch_nt<kSlope2, true, true>(a, n_events, perm, pairs_evaluated, stream);
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

}  // namespace retina
