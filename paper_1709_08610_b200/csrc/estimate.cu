// estimate.cu -- grid step (iv) ("for each cluster estimate track parameters"):
// per-peak sub-cell parameter estimate by 3-point quadratic interpolation along each axis
// (reading Z21).
//
// For a peak at cell c and axis i with both neighbours present, the parabola through
// (-1, R-), (0, R0), (+1, R+) peaks at
//     delta = (R- - R+) / (2 (R- - 2 R0 + R+)),
// and the estimate is theta_i = node_i[c_i] + delta * (node_i[c_i+1] - node_i[c_i-1]) / 2.
// A strict local maximum has R0 > R-, R0 > R+, so |delta| < 1/2 (the vertex stays in the cell);
// on a lattice boundary (a neighbour is missing) or a degenerate denominator the estimate
// falls back to the cell centre (delta = 0).  One thread per (event, peak slot).
#include "common.cuh"
#include "kernels.cuh"

namespace retina {

__global__ void __launch_bounds__(256) estimate_kernel(EstimateArgs a) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)a.n_events * a.capacity;
    if (gid >= total) return;
    const int e = (int)(gid / a.capacity), p = (int)(gid % a.capacity);
    const int P = a.P;
    if (p >= min(a.cnt[e], a.capacity)) return;
    const int n[3] = {a.n0, a.n1, a.n2};
    const int64_t cells = (int64_t)a.n0 * a.n1 * a.n2;
    const float *g = a.R + (int64_t)e * cells;
    const int c = a.idx[(int64_t)e * a.capacity + p];
    RETINA_ASSERT(c >= 0 && (int64_t)c < cells);
    // node indices in parameter order (tx, ty[, z0]); cell (i, j[, l]) at (l n0 + i) n1 + j (Z37)
    int ci[3];
    ci[1] = c % a.n1;
    ci[0] = (c / a.n1) % a.n0;
    ci[2] = c / (a.n0 * a.n1);
    const int stride[3] = {a.n1, 1, a.n0 * a.n1};
    const float r0 = __ldg(g + c);
    const float *nodes[3] = {a.nodes0, a.nodes1, a.nodes2};
    for (int i = 0; i < P; ++i) {
        const float t = __ldg(nodes[i] + ci[i]);
        float th = t;
        if (ci[i] > 0 && ci[i] < n[i] - 1) {
            const float rm = __ldg(g + c - stride[i]), rp = __ldg(g + c + stride[i]);
            const float den = __fmul_rn(2.f, __fadd_rn(__fsub_rn(rm, __fmul_rn(2.f, r0)), rp));
            if (den < 0.f) {
                float delta = __fdiv_rn(__fsub_rn(rm, rp), den);
                delta = fminf(fmaxf(delta, -0.5f), 0.5f);
                const float half = __fmul_rn(0.5f, __fsub_rn(__ldg(nodes[i] + ci[i] + 1), __ldg(nodes[i] + ci[i] - 1)));
                th = __fmaf_rn(delta, half, t);
            }
        }
        a.theta[((int64_t)e * a.capacity + p) * P + i] = th;
    }
}

cudaError_t launch_estimate(const EstimateArgs &a, cudaStream_t stream) {
    const int64_t total = (int64_t)a.n_events * a.capacity;
    if (total == 0) return cudaSuccess;
    const int64_t blocks = (total + 255) / 256;
    if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
    estimate_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace retina
