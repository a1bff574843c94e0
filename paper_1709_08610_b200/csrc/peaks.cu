// peaks.cu -- K2+K3: step (iii) as strict local maxima (Z6) and
// their ordered per-event compaction.
//
// One CTA per event sweeps the event's grid in chunks of 512 threads x 4 consecutive cells.
// A cell is flagged iff R_c >= threshold and R_c > R_n for every existing neighbour of its
// 3^P - 1 neighbourhood (short-circuit: most cells fail the threshold or the first
// neighbour, so the average cell reads ~2 values, mostly from L1/L2).  Flags are compacted
// with a warp-shuffle + shared-memory block scan, so peaks come out in ascending linear
// index with no atomics (bit-deterministic).  The running total is the TRUE count; only
// the first `capacity` entries are written.
#include "common.cuh"
#include "kernels.cuh"

namespace retina {

constexpr int kPeakThreads = 512;
constexpr int kPeakV = 4;

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

template <int P>
__device__ __forceinline__ bool is_peak(const float *__restrict__ g, int c, int n0, int n1, int n2,
                                        float thr) {
    const float v = __ldg(g + c);
    if (!(v >= thr)) return false;
    int l = 0, j, i;
    if (P == 3) {
        l = c % n2;
        const int t = c / n2;
        j = t % n1;
        i = t / n1;
    } else {
        j = c % n1;
        i = c / n1;
    }
    for (int di = -1; di <= 1; ++di) {
        const int ii = i + di;
        if (ii < 0 || ii >= n0) continue;
        for (int dj = -1; dj <= 1; ++dj) {
            const int jj = j + dj;
            if (jj < 0 || jj >= n1) continue;
            if (P == 3) {
                for (int dl = -1; dl <= 1; ++dl) {
                    const int ll = l + dl;
                    if (ll < 0 || ll >= n2 || (di == 0 && dj == 0 && dl == 0)) continue;
                    if (!(v > __ldg(g + ((ii * n1 + jj) * n2 + ll)))) return false;
                }
            } else {
                if (di == 0 && dj == 0) continue;
                if (!(v > __ldg(g + (ii * n1 + jj)))) return false;
            }
        }
    }
    return true;
}

template <int P>
__global__ void __launch_bounds__(kPeakThreads) find_peaks_kernel(PeakArgs a) {
    __shared__ int s_warp[kPeakThreads / 32];
    const int e = a.e_base + blockIdx.x;
    const int cells = a.n0 * a.n1 * a.n2;
    const float *g = a.R + (int64_t)e * cells;
    int32_t *oi = a.idx + (int64_t)e * a.capacity;
    float *ov = a.val + (int64_t)e * a.capacity;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int total = 0;
    for (int base = 0; base < cells; base += kPeakThreads * kPeakV) {
        const int c0 = base + threadIdx.x * kPeakV;
        unsigned mask = 0;
#pragma unroll
        for (int v = 0; v < kPeakV; ++v) {
            const int c = c0 + v;
            if (c < cells && is_peak<P>(g, c, a.n0, a.n1, a.n2, a.threshold)) mask |= 1u << v;
        }
        const int cnt = __popc(mask);
        const int incl = warp_incl_scan(cnt);
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int w = (lane < kPeakThreads / 32) ? s_warp[lane] : 0;
            w = warp_incl_scan(w);
            if (lane < kPeakThreads / 32) s_warp[lane] = w;
        }
        __syncthreads();
        int pos = total + incl - cnt + (warp > 0 ? s_warp[warp - 1] : 0);
        const int chunk_total = s_warp[kPeakThreads / 32 - 1];
#pragma unroll
        for (int v = 0; v < kPeakV; ++v) {
            if (mask & (1u << v)) {
                if (pos < a.capacity) {
                    oi[pos] = c0 + v;
                    ov[pos] = __ldg(g + c0 + v);
                }
                ++pos;
            }
        }
        total += chunk_total;
        __syncthreads();  // s_warp is rewritten by the next chunk
    }
    if (threadIdx.x == 0) a.cnt[e] = total;
}

cudaError_t launch_find_peaks(const PeakArgs &a0, int n_events, cudaStream_t stream) {
    for (int e0 = 0; e0 < n_events; e0 += 0x7fffffff) {
        PeakArgs a = a0;
        a.e_base = e0;
        const int ne = n_events - e0;
        if (a.P == 3)
            find_peaks_kernel<3><<<ne, kPeakThreads, 0, stream>>>(a);
        else
            find_peaks_kernel<2><<<ne, kPeakThreads, 0, stream>>>(a);
        const cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

}  // namespace retina
