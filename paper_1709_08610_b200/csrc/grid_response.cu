// grid_response.cu -- K1: Eq. (2) R_ij = sum_k exp(-s(x_k, theta_ij)^2 / sigma^2)
// (step (ii) PAPER.md:119) for every unit of every event.
//
// Mapping (K1):
//  * grid = (unit tiles, events); 256 threads = 8 warps per CTA.
//  * lanes run along the FASTEST axis of the response layout, so every warp store is one
//    128-byte line; each thread owns U units along a slower axis, so the part of the
//    residual that depends only on the lane's parameter (and the hit) is formed once per
//    (thread, hit) and reused U times.
//      LINE2D / SLOPE2: lanes over axis 1, U rows of axis 0.
//      SLOPE3:          the same within one z0 plane (layout [n2][n0][n1], Z37): the
//                       block's z0 node plays SLOPE2's z_ref, d = z - z0 formed exactly once per hit.
//  * the event's hits are staged in shared memory by TMA bulk copies (HitStage) and read
//    as warp-uniform LDS.128 broadcasts.
//  * per (unit, hit): residual by FMA (exact product), s^2, one FMUL by -log2(e)/sigma^2,
//    one MUFU.EX2, one FADD into a per-unit register accumulator (fixed order: hit array
//    order, so results are deterministic).
#include "common.cuh"
#include "kernels.cuh"

namespace retina {

template <int MODEL, int U, bool ZREF>
__global__ void __launch_bounds__(256) grid_response_kernel(GridArgs a) {
    extern __shared__ __align__(16) float4 s_hits[];
    __shared__ __align__(8) uint64_t s_bar[2];

    const int e = a.e_base + blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;

    HitStage st;
    st.init(s_hits, s_bar, a.hits + start, nh, a.cap);

    // fast-axis index (lanes: axis 1), first owned slow-axis index (axis 0), z0 plane (SLOPE3)
    const int tj = (a.n1 + 31) / 32, ti = (a.n0 + 8 * U - 1) / (8 * U);
    const int l = (MODEL == kSlope3) ? (int)(blockIdx.x / (tj * ti)) : 0;
    const int b = (MODEL == kSlope3) ? (int)(blockIdx.x % (tj * ti)) : (int)blockIdx.x;
    const int t_j = b % tj, t_i = b / tj;
    const int fast = t_j * 32 + lane, row0 = t_i * 8 * U + warp * U;
    const int nfast = a.n1, nslow = a.n0;
    const float pf = __ldg(a.nodes1 + min(fast, nfast - 1));
    float ps[U];
#pragma unroll
    for (int u = 0; u < U; ++u) ps[u] = __ldg(a.nodes0 + min(row0 + u, nslow - 1));
    const float negK = a.negK;
    constexpr bool EXACT_D = ZREF || MODEL == kSlope3;  // d = z - z_ref (or z - z0) as dh + dl
    const float zref = (MODEL == kSlope3) ? __ldg(a.nodes2 + l) : a.z_ref;

    float acc[U];
#pragma unroll
    for (int u = 0; u < U; ++u) acc[u] = 0.f;

    st.pass([&](const float4 *h, int len) {
#pragma unroll 2
        for (int k = 0; k < len; ++k) {
            const float4 hk = h[k];
            if (MODEL == kSlope2 || MODEL == kSlope3) {
                // lane parameter = ty (axis 1), rows = tx (axis 0)
                float sy, dh = hk.z, dl = 0.f;
                if (EXACT_D) {
                    two_sum(hk.z, -zref, dh, dl);
                    sy = __fmaf_rn(-pf, dl, __fmaf_rn(-pf, dh, hk.y));
                } else {
                    sy = __fmaf_rn(-pf, hk.z, hk.y);
                }
                const float sy2 = __fmul_rn(sy, sy);
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float sx = EXACT_D ? __fmaf_rn(-ps[u], dl, __fmaf_rn(-ps[u], dh, hk.x))
                                             : __fmaf_rn(-ps[u], hk.z, hk.x);
                    const float q = __fmaf_rn(sx, sx, sy2);
                    acc[u] = __fadd_rn(acc[u], ex2_approx(__fmul_rn(q, negK)));
                }
            } else {  // LINE2D: lane parameter = b (axis 1), rows = a (axis 0)
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    // r = y - a x as r_hi + r_lo (TwoProd + TwoSum), then s = (r_hi - b) + r_lo
                    const float p_hi = __fmul_rn(ps[u], hk.x);
                    const float p_lo = __fmaf_rn(ps[u], hk.x, -p_hi);
                    float r_hi, e1;
                    two_sum(hk.y, -p_hi, r_hi, e1);
                    const float r_lo = __fsub_rn(e1, p_lo);
                    const float s = __fadd_rn(__fsub_rn(r_hi, pf), r_lo);
                    const float q = __fmul_rn(s, s);
                    acc[u] = __fadd_rn(acc[u], ex2_approx(__fmul_rn(q, negK)));
                }
            }
        }
    });

    if (fast < nfast) {
        const int64_t cells = (int64_t)a.n0 * a.n1 * (MODEL == kSlope3 ? a.n2 : 1);
        float *out = a.R + (int64_t)e * cells + (int64_t)l * a.n0 * a.n1;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = row0 + u;
            if (r < nslow) out[(int64_t)r * a.n1 + fast] = acc[u];
        }
    }
}

template <int MODEL, int U, bool ZREF>
static cudaError_t launch_grid(const GridArgs &a0, int n_events, cudaStream_t stream) {
    auto kern = grid_response_kernel<MODEL, U, ZREF>;
    const size_t smem = (size_t)a0.cap * sizeof(float4);
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const long long tiles = (long long)((a0.n1 + 31) / 32) * ((a0.n0 + 8 * U - 1) / (8 * U)) *
                            (MODEL == kSlope3 ? a0.n2 : 1);
    if (tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        GridArgs a = a0;
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        kern<<<dim3((unsigned)tiles, ne), 256, smem, stream>>>(a);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

cudaError_t launch_grid_response(int model, const GridArgs &a, int n_events, cudaStream_t stream) {
    constexpr int U = 8;
    if (n_events == 0) return cudaSuccess;
    switch (model) {
        case kLine2D: return launch_grid<kLine2D, U, false>(a, n_events, stream);
        case kSlope2:
            return (a.z_ref == 0.f) ? launch_grid<kSlope2, U, false>(a, n_events, stream)
                                    : launch_grid<kSlope2, U, true>(a, n_events, stream);
        case kSlope3: return launch_grid<kSlope3, U, false>(a, n_events, stream);
    }
    return cudaErrorInvalidValue;
}

}  // namespace retina
