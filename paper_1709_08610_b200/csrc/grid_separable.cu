// grid_separable.cu -- K1s: Eq. (2) for the in-plane-distance models as a dense contraction.
//
// For SLOPE2 / SLOPE3 the squared in-plane distance splits into an x part that depends only
// on (tx, hit) and a y part that depends only on (ty, hit) (at fixed z0 for SLOPE3):
//     s^2 = (x - tx d)^2 + (y - ty d)^2,   d = z - z_ref (or z - z0),
// so the Gaussian of Eq. (1) factorises exactly, exp(-s^2/sigma^2) = e_x(tx, k) * e_y(ty, k),
// and the whole grid of Eq. (2) is a matrix product over the hit index k:
//     R[i][j] = sum_k EX[i][k] * EY[j][k],  EX[i][k] = 2^(-K (x_k - tx_i d_k)^2),
//                                           EY[j][k] = 2^(-K (y_k - ty_j d_k)^2).
// Each (unit, hit) pair is still evaluated -- as one FFMA of two Gaussian factors -- in the
// same hit order as the direct kernel, but the exps drop from n_tx*n_ty*N to (n_tx+n_ty)*N
// per 128x128 tile, so the kernel is bound by the FP32 FMA pipe (128 FMA/clk/SM) instead of
// MUFU (16 ex2/clk/SM).  All terms are positive, so the factorised sum has the same relative
// error as the direct one (no cancellation).
//
// Tiling: CTA = 256 threads computes a 128 (axis 0, tx) x 128 (axis 1, ty) tile of one event
// (and one z0 for SLOPE3).  Hits are staged in shared memory by TMA bulk copies (HitStage);
// per 32-hit chunk the CTA generates EX[32][128] and EY[32][128] into shared memory (one
// MUFU.EX2 each), then every thread accumulates an 8x8 register micro-tile with 32 FFMA2
// (row value broadcast) per 4 LDS.128.  (A variant that interleaved the next chunk's
// generation with this chunk's FFMA2s spilled at 128 registers and measured slower.)
#include "common.cuh"
#include "kernels.cuh"

namespace retina {

constexpr int SB_M = 128, SB_N = 128, SB_K = 32;

template <int MODEL, bool ZREF>
__global__ void __launch_bounds__(256, 2) grid_separable_kernel(GridArgs a) {
    extern __shared__ __align__(16) float4 s_hits[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ __align__(16) float sA[SB_K][SB_M];
    __shared__ __align__(16) float sB[SB_K][SB_N];

    const int e = a.e_base + blockIdx.y;
    const int tm = (a.n0 + SB_M - 1) / SB_M, tn = (a.n1 + SB_N - 1) / SB_N;
    int b = blockIdx.x;
    const int t_n = b % tn;
    b /= tn;
    const int t_m = b % tm;
    const int l = b / tm;  // z0 index (SLOPE3), 0 otherwise

    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;
    HitStage st;
    st.init(s_hits, s_bar, a.hits + start, nh, a.cap);

    const int tid = threadIdx.x;
    const int tr = tid >> 4, tc = tid & 15;  // compute roles: 16 x 16 threads, 8 x 8 each
    const int gi = tid & 127, gk = tid >> 7;  // generation roles: unit gi, hits gk + 2m
    const float pa = __ldg(a.nodes0 + min(t_m * SB_M + gi, a.n0 - 1));  // tx
    const float pb = __ldg(a.nodes1 + min(t_n * SB_N + gi, a.n1 - 1));  // ty
    const float z0 = (MODEL == kSlope3) ? __ldg(a.nodes2 + l) : a.z_ref;
    const float negK = a.negK;

    // 8 x 8 micro-tile as 8 x 4 column PAIRS: one FFMA2 (row value broadcast to both halves)
    // updates two units, halving issue slots; each half is an IEEE fma.rn, same as FFMA.
    float2 acc[8][4];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = make_float2(0.f, 0.f);

    st.pass([&](const float4 *h, int len) {
        for (int k0 = 0; k0 < len; k0 += SB_K) {
#pragma unroll 4
            for (int m = 0; m < SB_K / 2; ++m) {
                const int k = gk + 2 * m;
                float ea = 0.f, eb = 0.f;
                if (k0 + k < len) {
                    const float4 hk = h[k0 + k];
                    float sx, sy;
                    if (MODEL == kSlope3 || ZREF) {
                        float dh, dl;
                        two_sum(hk.z, -z0, dh, dl);  // d = z - z0 exactly as dh + dl
                        sx = __fmaf_rn(-pa, dl, __fmaf_rn(-pa, dh, hk.x));
                        sy = __fmaf_rn(-pb, dl, __fmaf_rn(-pb, dh, hk.y));
                    } else {
                        sx = __fmaf_rn(-pa, hk.z, hk.x);
                        sy = __fmaf_rn(-pb, hk.z, hk.y);
                    }
                    ea = ex2_approx(__fmul_rn(__fmul_rn(sx, sx), negK));
                    eb = ex2_approx(__fmul_rn(__fmul_rn(sy, sy), negK));
                }
                sA[k][gi] = ea;
                sB[k][gi] = eb;
            }
            __syncthreads();
#pragma unroll 8
            for (int k = 0; k < SB_K; ++k) {
                const float4 a0 = *reinterpret_cast<const float4 *>(&sA[k][tr * 4]);
                const float4 a1 = *reinterpret_cast<const float4 *>(&sA[k][64 + tr * 4]);
                const float4 b0 = *reinterpret_cast<const float4 *>(&sB[k][tc * 4]);
                const float4 b1 = *reinterpret_cast<const float4 *>(&sB[k][64 + tc * 4]);
                const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                const float2 bv[4] = {make_float2(b0.x, b0.y), make_float2(b0.z, b0.w), make_float2(b1.x, b1.y),
                                      make_float2(b1.z, b1.w)};
#pragma unroll
                for (int r = 0; r < 8; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        acc[r][c] = __ffma2_rn(make_float2(av[r], av[r]), bv[c], acc[r][c]);
            }
            __syncthreads();
        }
    });

#define ACC(r, c) (((c) & 1) ? acc[r][(c) >> 1].y : acc[r][(c) >> 1].x)
    const int64_t cells = (int64_t)a.n0 * a.n1 * (MODEL == kSlope3 ? a.n2 : 1);
    float *out = a.R + (int64_t)e * cells + (int64_t)l * a.n0 * a.n1;  // z0 plane l (Z37)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int i = t_m * SB_M + (r < 4 ? tr * 4 + r : 64 + tr * 4 + r - 4);
        if (i >= a.n0) continue;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            const int j0 = t_n * SB_N + half * 64 + tc * 4;
            {
                float *p = out + (int64_t)i * a.n1 + j0;
                if (j0 + 3 < a.n1 && ((reinterpret_cast<uintptr_t>(p) & 15u) == 0)) {
                    *reinterpret_cast<float4 *>(p) =
                        make_float4(ACC(r, half * 4), ACC(r, half * 4 + 1), ACC(r, half * 4 + 2), ACC(r, half * 4 + 3));
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        if (j0 + c < a.n1) p[c] = ACC(r, half * 4 + c);
                }
            }
        }
    }
}

#undef ACC

template <int MODEL, bool ZREF>
static cudaError_t launch_sep(const GridArgs &a0, int n_events, cudaStream_t stream) {
    auto kern = grid_separable_kernel<MODEL, ZREF>;
    const size_t smem = (size_t)a0.cap * sizeof(float4);
    cudaError_t err = ensure_dynamic_smem(kern, smem);
    if (err != cudaSuccess) return err;
    const long long tiles = (long long)((a0.n0 + SB_M - 1) / SB_M) * ((a0.n1 + SB_N - 1) / SB_N) *
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

cudaError_t launch_grid_separable(int model, const GridArgs &a, int n_events, cudaStream_t stream) {
    if (n_events == 0) return cudaSuccess;
    switch (model) {
        case kSlope2:
            return (a.z_ref == 0.f) ? launch_sep<kSlope2, false>(a, n_events, stream)
                                    : launch_sep<kSlope2, true>(a, n_events, stream);
        case kSlope3: return launch_sep<kSlope3, false>(a, n_events, stream);
    }
    return cudaErrorInvalidValue;  // LINE2D does not factorise: use the direct kernel
}

}  // namespace retina
