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
// Consecutive cells per thread per sweep: 16 (four float4 loads in flight) for P = 2; 4 for P = 3,
// whose wider peaks put more cells above threshold, each with 26 neighbour reads, so fewer cells per
// thread keep the warps balanced (cfg4 peaks 22 ms with 4 vs 78 with 16; cfg3 9.5 with 16 vs 15 with 4).
template <int P>
struct PeakV {
    static constexpr int v = (P == 3) ? 4 : 16;
};
constexpr int kSlabCells = 131072;  // cells per CTA in the workspace (two-pass) variant
#ifndef RETINA_PK_SLABLIST
#define RETINA_PK_SLABLIST 1024  // (256: the dense-hit cfg3 variant rescanned most slabs, 6.2 vs 4.5 ms per 1,024 events)
#endif
constexpr int kSlabList = RETINA_PK_SLABLIST;  // peaks a slab keeps from pass 1 (more: pass 2 rescans it)

__device__ __forceinline__ int warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Neighbour test of cell c whose value v (>= threshold) is already loaded.
template <int P>
__device__ __forceinline__ bool beats_neighbours(const float *__restrict__ g, int c, float v, int n0, int n1,
                                                 int n2) {
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
__device__ __forceinline__ bool is_peak(const float *__restrict__ g, int c, int n0, int n1, int n2,
                                        float thr) {
    const float v = __ldg(g + c);
    return v >= thr && beats_neighbours<P>(g, c, v, n0, n1, n2);
}

// Flags and (when WRITE) compacts the peaks of cells [c_begin, c_end) of one event, writing the
// i-th peak found at output position pos0 + i.  Returns the number of peaks in the range.
template <int P, bool WRITE>
__device__ __forceinline__ int scan_range(const PeakArgs &a, const float *g, int32_t *oi, float *ov, int c_begin,
                                          int c_end, int pos0, int *s_warp, int cap) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int total = 0;
    constexpr int kPeakV = PeakV<P>::v;
    for (int base = c_begin; base < c_end; base += kPeakThreads * kPeakV) {
        const int c0 = base + threadIdx.x * kPeakV;
        unsigned mask = 0;
        if (c0 + kPeakV <= c_end && ((reinterpret_cast<uintptr_t>(g + c0) & 15u) == 0)) {
            // 16-byte loads for the thread's cells, all in flight together (most cells fail the
            // threshold right here)
            float vv[kPeakV];
#pragma unroll
            for (int u = 0; u < kPeakV; u += 4) {
                const float4 q = __ldg(reinterpret_cast<const float4 *>(g + c0 + u));
                vv[u] = q.x;
                vv[u + 1] = q.y;
                vv[u + 2] = q.z;
                vv[u + 3] = q.w;
            }
            // neighbours along the fastest axis that are the thread's own cells are compared first,
            // from registers: a candidate on a slope along that axis is rejected with no load
            const int nlast = (P == 3) ? a.n2 : a.n1;
#pragma unroll
            for (int v = 0; v < kPeakV; ++v) {
                if (!(vv[v] >= a.threshold)) continue;
                const int pos = (c0 + v) % nlast;  // position along the fastest axis (rows may wrap)
                if (v > 0 && pos > 0 && !(vv[v] > vv[v - 1])) continue;
                if (v + 1 < kPeakV && pos + 1 < nlast && !(vv[v] > vv[v + 1])) continue;
                if (beats_neighbours<P>(g, c0 + v, vv[v], a.n0, a.n1, a.n2)) mask |= 1u << v;
            }
        } else {
#pragma unroll
            for (int v = 0; v < kPeakV; ++v) {
                const int c = c0 + v;
                if (c < c_end && is_peak<P>(g, c, a.n0, a.n1, a.n2, a.threshold)) mask |= 1u << v;
            }
        }
        const int cnt = __popc(mask);
        // most sweeps hold no peak: one barrier decides that, and the block scan is skipped
        if (!__syncthreads_or(cnt != 0)) continue;
        const int incl = warp_incl_scan(cnt);
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int w = (lane < kPeakThreads / 32) ? s_warp[lane] : 0;
            w = warp_incl_scan(w);
            if (lane < kPeakThreads / 32) s_warp[lane] = w;
        }
        __syncthreads();
        if (WRITE) {
            int pos = pos0 + total + incl - cnt + (warp > 0 ? s_warp[warp - 1] : 0);
#pragma unroll
            for (int v = 0; v < kPeakV; ++v) {
                if (mask & (1u << v)) {
                    if (pos < cap) {
                        oi[pos] = c0 + v;
                        ov[pos] = __ldg(g + c0 + v);
                    }
                    ++pos;
                }
            }
        }
        total += s_warp[kPeakThreads / 32 - 1];
        __syncthreads();  // s_warp is rewritten by the next chunk
    }
    return total;
}

// Single pass, one CTA per event (no workspace).
template <int P>
__global__ void __launch_bounds__(kPeakThreads) find_peaks_kernel(PeakArgs a) {
    __shared__ int s_warp[kPeakThreads / 32];
    const int e = a.e_base + blockIdx.x;
    const int cells = a.n0 * a.n1 * a.n2;
    const float *g = a.R + (int64_t)e * cells;
    const int total = scan_range<P, true>(a, g, a.idx + (int64_t)e * a.capacity, a.val + (int64_t)e * a.capacity,
                                          0, cells, 0, s_warp, a.capacity);
    if (threadIdx.x == 0) a.cnt[e] = total;
}

// Two passes over slabs of kSlabCells cells, grid (slabs, events), with a caller-owned
// workspace: int32 counts [events][slabs], then per slab a list of its first kSlabList peaks
// (int32 index [events][slabs][kSlabList], fp32 value [events][slabs][kSlabList]).
// (1) each slab scans its cells once, counts its peaks and keeps the first kSlabList of them
// (ascending index); (2) each slab sums the counts of the slabs before it (fixed order:
// deterministic) and copies its list to that offset -- only a slab with more than kSlabList
// peaks scans its cells again.  The last slab writes the event's true count.  Same output as
// the single pass, many CTAs per event, and (for sparse peaks) one read of the grid.
struct SlabWs {
    int32_t *count;
    int32_t *idx;
    float *val;
    __device__ __forceinline__ static SlabWs at(int32_t *ws, int n_ev, int n_slabs) {
        SlabWs w;
        const int64_t lists = (int64_t)n_ev * n_slabs;
        w.count = ws;
        w.idx = ws + lists;
        w.val = reinterpret_cast<float *>(ws + lists + lists * kSlabList);
        return w;
    }
};

template <int P>
__global__ void __launch_bounds__(kPeakThreads) count_peaks_slab_kernel(PeakArgs a, int32_t *ws, int n_slabs) {
    __shared__ int s_warp[kPeakThreads / 32];
    const int e = a.e_base + blockIdx.y, b = blockIdx.x;
    const int cells = a.n0 * a.n1 * a.n2;
    const int c_begin = b * kSlabCells, c_end = min(cells, c_begin + kSlabCells);
    const SlabWs w = SlabWs::at(ws, gridDim.y, n_slabs);
    const int64_t slab = (int64_t)blockIdx.y * n_slabs + b;
    const int n = scan_range<P, true>(a, a.R + (int64_t)e * cells, w.idx + slab * kSlabList,
                                      w.val + slab * kSlabList, c_begin, c_end, 0, s_warp, kSlabList);
    if (threadIdx.x == 0) w.count[slab] = n;
}

template <int P>
__global__ void __launch_bounds__(kPeakThreads) write_peaks_slab_kernel(PeakArgs a, const int32_t *ws, int n_slabs) {
    __shared__ int s_warp[kPeakThreads / 32];
    __shared__ int s_off;
    const int e = a.e_base + blockIdx.y, b = blockIdx.x;
    const int cells = a.n0 * a.n1 * a.n2;
    const SlabWs w = SlabWs::at(const_cast<int32_t *>(ws), gridDim.y, n_slabs);
    const int32_t *cnt = w.count + (int64_t)blockIdx.y * n_slabs;
    if (threadIdx.x == 0) {
        int off = 0;
        for (int i = 0; i < b; ++i) off += cnt[i];
        s_off = off;
    }
    __syncthreads();
    const int off = s_off, n = cnt[b];
    int32_t *oi = a.idx + (int64_t)e * a.capacity;
    float *ov = a.val + (int64_t)e * a.capacity;
    if (off < a.capacity) {
        if (n <= kSlabList) {  // pass 1 kept every peak of this slab: copy, no grid read
            const int64_t slab = (int64_t)blockIdx.y * n_slabs + b;
            const int m = min(n, a.capacity - off);
            for (int i = threadIdx.x; i < m; i += kPeakThreads) {
                oi[off + i] = w.idx[slab * kSlabList + i];
                ov[off + i] = w.val[slab * kSlabList + i];
            }
        } else {
            const int c_begin = b * kSlabCells, c_end = min(cells, c_begin + kSlabCells);
            scan_range<P, true>(a, a.R + (int64_t)e * cells, oi, ov, c_begin, c_end, off, s_warp, a.capacity);
        }
    }
    if (b == n_slabs - 1 && threadIdx.x == 0) a.cnt[e] = off + n;
}

cudaError_t launch_find_peaks(const PeakArgs &a0, int n_events, cudaStream_t stream) {
    PeakArgs a = a0;
    a.e_base = 0;
    if (a.P == 3)
        find_peaks_kernel<3><<<n_events, kPeakThreads, 0, stream>>>(a);
    else
        find_peaks_kernel<2><<<n_events, kPeakThreads, 0, stream>>>(a);
    return cudaGetLastError();
}

int peaks_slabs(int cells) { return (cells + kSlabCells - 1) / kSlabCells; }

size_t peaks_workspace_bytes(long long n_events, int P, int n0, int n1, int n2) {
    if (P == 3 && peaks3_brick_ok(n0, n1, n2)) return peaks3_workspace_bytes(n_events, n0, n1, n2);
    const long long lists = n_events * peaks_slabs(n0 * n1 * n2);
    return (size_t)lists * (sizeof(int32_t) + (size_t)kSlabList * (sizeof(int32_t) + sizeof(float)));
}

cudaError_t launch_find_peaks_ws(const PeakArgs &a0, int n_events, int32_t *ws, cudaStream_t stream) {
    if (a0.P == 3 && peaks3_brick_ok(a0.n0, a0.n1, a0.n2))  // plane blocks staged by TMA (peaks3.cu)
        return launch_find_peaks3_brick(a0, n_events, ws, stream);
    const int cells = a0.n0 * a0.n1 * a0.n2;
    const int n_slabs = peaks_slabs(cells);
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        PeakArgs a = a0;
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        const dim3 grid(n_slabs, ne);
        if (a.P == 3) {
            count_peaks_slab_kernel<3><<<grid, kPeakThreads, 0, stream>>>(a, ws, n_slabs);
            write_peaks_slab_kernel<3><<<grid, kPeakThreads, 0, stream>>>(a, ws, n_slabs);
        } else {
            count_peaks_slab_kernel<2><<<grid, kPeakThreads, 0, stream>>>(a, ws, n_slabs);
            write_peaks_slab_kernel<2><<<grid, kPeakThreads, 0, stream>>>(a, ws, n_slabs);
        }
        const cudaError_t err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

}  // namespace retina
