// cull.cuh -- exact-zero pair culling shared by K4c (multistart.cu) and K6c (newton.cu).
//
// With ex2.approx.ftz, w = 2^(-K s^2 log2 e) is +0 whenever the exponent is below -126 (the
// result would be subnormal and is flushed), and a +0 weight leaves R, the gradient sums and the
// Hessian sums unchanged bit for bit.  A warp may therefore skip every hit that a conservative
// bound puts beyond K s^2 > 128 for ALL of its parameter points (room for fp32 rounding of s and
// of the exponent), visiting the rest in the original hit order with unchanged arithmetic.
#pragma once
#include "common.cuh"
#include "kernels.cuh"

#include <type_traits>

namespace retina {

struct McBox {
    float lo[3], hi[3];  // the seeds' parameter box; lo[0] > hi[0]: empty
};

// the box of the warp's valid seeds (warp-uniform)
template <int P, int S>
__device__ __forceinline__ McBox mc_warp_box(const float (&th)[S][3], const bool (&ok)[S]) {
    McBox b;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        b.lo[i] = 3.4e38f;
        b.hi[i] = -3.4e38f;
    }
#pragma unroll
    for (int s = 0; s < S; ++s)
        if (ok[s])
#pragma unroll
            for (int i = 0; i < P; ++i) {
                b.lo[i] = fminf(b.lo[i], th[s][i]);
                b.hi[i] = fmaxf(b.hi[i], th[s][i]);
            }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < P; ++i) {
            b.lo[i] = fminf(b.lo[i], __shfl_xor_sync(0xffffffffu, b.lo[i], o));
            b.hi[i] = fmaxf(b.hi[i], __shfl_xor_sync(0xffffffffu, b.hi[i], o));
        }
    return b;
}

// least |x - t d| over t in [t0, t1] and d in [d0, d1] (0 when the range of t d contains x)
__device__ __forceinline__ float mc_min_abs(float x, float t0, float t1, float d0, float d1) {
    const float p00 = t0 * d0, p01 = t0 * d1, p10 = t1 * d0, p11 = t1 * d1;
    const float pmin = fminf(fminf(p00, p01), fminf(p10, p11)), pmax = fmaxf(fmaxf(p00, p01), fmaxf(p10, p11));
    // rounded products: widen the range by 1e-6 of its magnitude so it holds every exact t d
    const float slack = 1e-6f * fmaxf(fabsf(pmin), fabsf(pmax));
    const float lo = x - (pmax + slack), hi = x - (pmin - slack);  // s ranges over [lo, hi]
    return (lo > 0.f) ? lo : (hi < 0.f ? -hi : 0.f);
}

// The warp's list of hits within reach of the box B: hit k is kept unless, for every parameter
// tuple in B, K ((x - tx d)^2 + (y - ty d)^2) > 128 (then every seed inside B has an ex2 argument
// < -126, with room for fp32 rounding: w = +0 exactly); d = z - z_ref (SLOPE2) or z - z0 over the
// box's z0 range (SLOPE3).  In hit order; returns the length.
// (mc_build_list_range: the hits kb .. n - 1 only; T = float4 lists copies of the hits.)
template <int MODEL, bool ZREF, class T>
__device__ __forceinline__ int mc_build_list_range(const float4 *h, int kb, int n, const McBox &B, float K, float zref,
                                                   T *list) {
    const int lane = threadIdx.x & 31;
    if (B.lo[0] > B.hi[0]) return 0;  // no valid seed in this warp
    int L = 0;
    for (int k0 = kb; k0 < n; k0 += 32) {
        const int k = k0 + lane;
        bool keep = false;
        if (k < n && MODEL == kSlope2 && !ZREF) {
            // d = z exactly: s_x = x - tx z ranges over [x - hi z, x - lo z] (z >= 0; swapped for
            // z < 0), so min |s_x| = max(0, x - hi z, lo z - x), each term one FMA (within half an
            // ulp of the exact value; the 0.99999 below covers it)
            const float4 hk = h[k];
            const bool pos = hk.z >= 0.f;
            const float ax = pos ? B.hi[0] : B.lo[0], bx = pos ? B.lo[0] : B.hi[0];
            const float ay = pos ? B.hi[1] : B.lo[1], by = pos ? B.lo[1] : B.hi[1];
            const float mx = fmaxf(0.f, fmaxf(__fmaf_rn(-ax, hk.z, hk.x), __fmaf_rn(bx, hk.z, -hk.x)));
            const float my = fmaxf(0.f, fmaxf(__fmaf_rn(-ay, hk.z, hk.y), __fmaf_rn(by, hk.z, -hk.y)));
            keep = K * __fmaf_rn(mx, mx, my * my) * 0.99999f <= 128.f;
        } else if (k < n) {
            const float4 hk = h[k];
            float d0, d1;  // the range of d, rounded outwards
            if (MODEL == kSlope3) {
                d0 = __fsub_rd(hk.z, B.hi[2]);
                d1 = __fsub_ru(hk.z, B.lo[2]);
            } else {
                d0 = ZREF ? __fsub_rd(hk.z, zref) : hk.z;
                d1 = ZREF ? __fsub_ru(hk.z, zref) : hk.z;
            }
            const float mx = mc_min_abs(hk.x, B.lo[0], B.hi[0], d0, d1);
            const float my = mc_min_abs(hk.y, B.lo[1], B.hi[1], d0, d1);
            keep = K * __fmaf_rn(mx, mx, my * my) * 0.99999f <= 128.f;
        }
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            if constexpr (std::is_same<T, float4>::value)
                list[L + __popc(b & ((1u << lane) - 1u))] = h[k];  // a copy of the hit (K6c)
            else
                list[L + __popc(b & ((1u << lane) - 1u))] = (uint16_t)k;
        }
        L += __popc(b);
    }
    __syncwarp();
    return L;
}

template <int MODEL, bool ZREF>
__device__ __forceinline__ int mc_build_list(const float4 *h, int n, const McBox &B, float K, float zref,
                                             uint16_t *list) {
    return mc_build_list_range<MODEL, ZREF>(h, 0, n, B, K, zref, list);
}

}  // namespace retina
