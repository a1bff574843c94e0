// multistart.cu -- K4: Algorithm 1's update loop with update = fixed-step
// gradient ascent clamped to the prior box (Z7):
//     theta^{j+1} = clamp(theta^j + step * grad R(theta^j)),  j < n_iters,
// then R(theta^n) and (optionally) grad R(theta^n).
//
// Mapping (K4): grid = (seed blocks, events), 128 threads per CTA, each thread
// owns S = 2 seeds (lanes over consecutive seeds: coalesced seed loads / stores).  The event's
// hits are staged ONCE in shared memory by a TMA bulk copy and stay resident for all
// n_iters + 1 passes when they fit (HitStage); otherwise they stream per pass.  Each pass
// accumulates, per seed, R = sum w and the raw gradient sums in registers, in hit-array order;
// the 2/sigma^2 factor is applied once per seed.
//
// Gradient (chain rule through s^2):
//   LINE2D  s = y - a x - b:           dR/da = c2 sum w s x,   dR/db = c2 sum w s
//   SLOPE2  s = (x - tx d, y - ty d):  dR/dtx = c2 sum w s_x d, dR/dty = c2 sum w s_y d
//   SLOPE3  d = z - z0:                ... and dR/dz0 = -c2 (tx sum w s_x + ty sum w s_y)
// with w = exp(-s^2/sigma^2) = ex2(-K s^2), c2 = 2/sigma^2.
#include "common.cuh"
#include "kernels.cuh"

namespace retina {

constexpr int kMsThreads = 128;

template <int MODEL, int S, bool ZREF, bool GRAD>
__device__ __forceinline__ void ms_pass(HitStage &st, const float (&th)[S][3], float negK, float zref,
                                        float (&R)[S], float (&G)[S][4]) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
        R[s] = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) G[s][i] = 0.f;
    }
    float dh[S], dl[S];
    float zprev = __int_as_float(0x7fc00000);  // NaN: the first hit always re-forms d
    st.pass([&](const float4 *h, int len) {
#pragma unroll 2
        for (int k = 0; k < len; ++k) {
            const float4 hk = h[k];
            if (MODEL == kSlope2) {
                float hdh = hk.z, hdl = 0.f;
                if (ZREF) two_sum(hk.z, -zref, hdh, hdl);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    float sx, sy;
                    if (ZREF) {
                        sx = __fmaf_rn(-th[s][0], hdl, __fmaf_rn(-th[s][0], hdh, hk.x));
                        sy = __fmaf_rn(-th[s][1], hdl, __fmaf_rn(-th[s][1], hdh, hk.y));
                    } else {
                        sx = __fmaf_rn(-th[s][0], hk.z, hk.x);
                        sy = __fmaf_rn(-th[s][1], hk.z, hk.y);
                    }
                    const float q = __fmaf_rn(sx, sx, __fmul_rn(sy, sy));
                    const float w = ex2_approx(__fmul_rn(q, negK));
                    R[s] = __fadd_rn(R[s], w);
                    if (GRAD) {
                        const float wd = __fmul_rn(w, hdh);
                        G[s][0] = __fmaf_rn(wd, sx, G[s][0]);
                        G[s][1] = __fmaf_rn(wd, sy, G[s][1]);
                    }
                }
            } else if (MODEL == kSlope3) {
                if (hk.z != zprev) {  // warp-uniform: every thread reads the same hit
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
                        const float wd = __fmul_rn(w, dh[s]);
                        G[s][0] = __fmaf_rn(wd, sx, G[s][0]);
                        G[s][1] = __fmaf_rn(wd, sy, G[s][1]);
                        G[s][2] = __fmaf_rn(w, sx, G[s][2]);
                        G[s][3] = __fmaf_rn(w, sy, G[s][3]);
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

template <int MODEL, int S, bool ZREF>
__global__ void __launch_bounds__(kMsThreads) multistart_kernel(MultistartArgs a) {
    extern __shared__ __align__(16) float4 s_hits[];
    __shared__ __align__(8) uint64_t s_bar[2];
    constexpr int P = (MODEL == kSlope3) ? 3 : 2;

    const int e = a.e_base + blockIdx.y;
    const int start = a.offsets[e], nh = a.offsets[e + 1] - start;
    HitStage st;
    st.init(s_hits, s_bar, a.hits + start, nh, a.cap);

    int sid[S];
    float th[S][3];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        sid[s] = blockIdx.x * (kMsThreads * S) + s * kMsThreads + threadIdx.x;
        const int64_t src = ((int64_t)e * a.n_seeds + min(sid[s], a.n_seeds - 1)) * P;
#pragma unroll
        for (int i = 0; i < 3; ++i) th[s][i] = (i < P) ? __ldg(a.seeds + src + i) : 0.f;
    }

    float R[S], G[S][4], g[S][3];
    for (int it = 0; it < a.n_iters; ++it) {
        ms_pass<MODEL, S, ZREF, true>(st, th, a.negK, a.z_ref, R, G);
        ms_gradient<MODEL, S>(th, G, a.c2, g);
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int i = 0; i < P; ++i)
                th[s][i] = fminf(fmaxf(__fmaf_rn(a.step, g[s][i], th[s][i]), a.lo[i]), a.hi[i]);
    }
    if (a.grad_out) {
        ms_pass<MODEL, S, ZREF, true>(st, th, a.negK, a.z_ref, R, G);
        ms_gradient<MODEL, S>(th, G, a.c2, g);
    } else {
        ms_pass<MODEL, S, ZREF, false>(st, th, a.negK, a.z_ref, R, G);
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

template <int MODEL, bool ZREF>
static cudaError_t launch_ms(const MultistartArgs &a0, int n_events, cudaStream_t stream) {
    constexpr int S = 2;
    auto kern = multistart_kernel<MODEL, S, ZREF>;
    const size_t smem = (size_t)a0.cap * sizeof(float4);
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const int blocks = (a0.n_seeds + kMsThreads * S - 1) / (kMsThreads * S);
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        MultistartArgs a = a0;
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        kern<<<dim3(blocks, ne), kMsThreads, smem, stream>>>(a);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
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

}  // namespace retina
