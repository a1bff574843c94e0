// pack.cu -- K8: the per-rank result record of the one gather (
// north star "one NCCL gather over NVLink for found tracks and timings only").
//
// Layout (32-bit words; float fields are stored as their bit patterns, so the buffer is
// exact and dtype-agnostic for the collective):
//   header [RETINA_PACK_HEADER]: rank, event_base, n_events, peaks_total, tracks_total,
//                                pairs_grid / 1e9 (f32), pairs_multistart / 1e9 (f32), 0
//   per event [2 + 2 keep + keep (P + 2)]:
//     n_peaks, n_tracks (TRUE counts), keep x peak index (-1 past the count),
//     keep x peak value (f32, 0 past the count), keep x (theta[P] f32, R f32, size) (0 past the count)
// Two kernels: the records (one thread per word, grid-stride) and the header totals (one
// CTA, integer sums: deterministic).
#include "../../include/retina.h"
#include "kernels.cuh"

namespace retina {

__global__ void pack_records_kernel(PackArgs a) {
    const int W = 2 + 2 * a.keep + a.keep * (a.P + 2);
    const long long total = (long long)a.n_events * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int e = (int)(i / W);
        int w = (int)(i - (long long)e * W);
        uint32_t v;
        const int pc = a.peak_count[e], tc = a.track_count[e];
        if (w == 0) {
            v = (uint32_t)pc;
        } else if (w == 1) {
            v = (uint32_t)tc;
        } else if ((w -= 2) < a.keep) {  // peak index
            v = (w < pc && w < a.peak_cap) ? (uint32_t)a.peak_index[(long long)e * a.peak_cap + w] : 0xffffffffu;
        } else if ((w -= a.keep) < a.keep) {  // peak value
            v = (w < pc && w < a.peak_cap) ? __float_as_uint(a.peak_value[(long long)e * a.peak_cap + w]) : 0u;
        } else {  // track k, field f
            w -= a.keep;
            const int k = w / (a.P + 2), f = w - k * (a.P + 2);
            if (k < tc && k < a.track_cap) {
                const long long t = (long long)e * a.track_cap + k;
                v = (f < a.P) ? __float_as_uint(a.track_theta[t * a.P + f])
                              : (f == a.P) ? __float_as_uint(a.track_response[t]) : (uint32_t)a.track_size[t];
            } else {
                v = 0u;
            }
        }
        a.out[RETINA_PACK_HEADER + i] = v;
    }
}

__global__ void pack_header_kernel(PackArgs a) {
    __shared__ unsigned long long sp[32], st[32];
    unsigned long long p = 0, t = 0;
    for (int e = threadIdx.x; e < a.n_events; e += blockDim.x) {
        p += (unsigned long long)a.peak_count[e];
        t += (unsigned long long)a.track_count[e];
    }
    for (int o = 16; o > 0; o >>= 1) {
        p += __shfl_xor_sync(0xffffffffu, p, o);
        t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    if ((threadIdx.x & 31) == 0) {
        sp[threadIdx.x >> 5] = p;
        st[threadIdx.x >> 5] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        p = t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            p += sp[w];
            t += st[w];
        }
        for (int i = 0; i < RETINA_PACK_HEADER; ++i) a.out[i] = a.header[i];
        a.out[3] = (uint32_t)(p > 0xffffffffull ? 0xffffffffull : p);
        a.out[4] = (uint32_t)(t > 0xffffffffull ? 0xffffffffull : t);
    }
}

cudaError_t launch_pack(const PackArgs &a, cudaStream_t stream) {
    const long long W = 2 + 2 * a.keep + (long long)a.keep * (a.P + 2);
    const long long total = (long long)a.n_events * W;
    if (total > 0) {
        const long long want = (total + 255) / 256;
        const int blocks = (int)(want < 148 * 16 ? want : 148 * 16);
        pack_records_kernel<<<blocks, 256, 0, stream>>>(a);
        cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    pack_header_kernel<<<1, 1024, 0, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace retina
