// merge.cu -- K5: Algorithm 1 "cluster solutions {theta^q_i}; for each cluster select solution
// with highest response and above threshold R0", Z9/Z10:
//   keep seeds with R >= R0; order by (R desc, theta lexicographic asc, seed index asc);
//   scan: a seed joins the EARLIEST-created leader within the per-axis Chebyshev radius
//   (differences in fp64, exact for fp32 inputs), else it founds a new leader.
//
// One CTA (512 threads) per event:
//   1. ordered compaction of the above-threshold seeds into 64-bit keys
//      (hi = order-reversed R bits, lo = seed index), block scan, no atomics;
//   2. bitonic sort of the keys in shared memory; exact R ties fall back to the theta
//      lexicographic comparison (loaded from global) and then to the seed index, so the
//      order is total and matches the oracle's comparator;
//   3. the greedy scan in rounds of 32 candidates: all 16 warps match the round's candidates
//      against the leaders founded before the round (smallest index per candidate), then warp 0
//      settles the round in order against the leaders founded within it.  Leader records
//      (size << 32 | seed) overwrite key slots that have already been consumed (leader l is
//      founded by an item at position >= l).
#include "common.cuh"
#include "kernels.cuh"

namespace retina {

constexpr int kMergeThreads = 512;
constexpr int kLeaderCache = 1024;

__device__ __forceinline__ int warp_incl_scan_m(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

__device__ __forceinline__ uint32_t desc_key(float r) {
    uint32_t u = __float_as_uint(r);
    if ((u << 1) == 0) u = 0;  // -0 == +0
    const uint32_t ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);  // ascending-order map
    return ~ord;                                                        // descending R
}

__device__ __forceinline__ bool key_less(uint64_t a, uint64_t b, const float *__restrict__ th, int P) {
    const uint32_t ha = (uint32_t)(a >> 32), hb = (uint32_t)(b >> 32);
    if (ha != hb) return ha < hb;
    if (ha == 0xffffffffu) return false;  // padding
    const int ia = (int)(uint32_t)a, ib = (int)(uint32_t)b;
    for (int i = 0; i < P; ++i) {
        const float ta = __ldg(th + (int64_t)ia * P + i), tb = __ldg(th + (int64_t)ib * P + i);
        if (ta < tb) return true;
        if (ta > tb) return false;
    }
    return ia < ib;
}

__global__ void __launch_bounds__(kMergeThreads) merge_kernel(MergeArgs a) {
    extern __shared__ __align__(16) uint64_t s_key[];
    __shared__ int s_warp[kMergeThreads / 32];
    __shared__ float s_lt[kLeaderCache * 3];
    __shared__ int s_m;
    __shared__ int s_csid[32], s_cmin[32];  // the round's candidates: seed, smallest matching old leader
    __shared__ float s_ct[32 * 3];           // the round's candidates: theta

    const int e = a.e_base + blockIdx.x;
    const int P = a.P, n = a.n_seeds;
    const float *th = a.theta + (int64_t)e * n * P;
    const float *rr = a.R + (int64_t)e * n;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double r0 = a.radius[0], r1 = a.radius[1], r2 = a.radius[2];

    // 1. ordered compaction of R >= threshold
    int total = 0;
    for (int base = 0; base < n; base += kMergeThreads) {
        const int s = base + threadIdx.x;
        float r = 0.f;
        const bool keep = (s < n) && ((r = __ldg(rr + s)) >= a.threshold);
        const int incl = warp_incl_scan_m(keep ? 1 : 0);
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            int w = (lane < kMergeThreads / 32) ? s_warp[lane] : 0;
            w = warp_incl_scan_m(w);
            if (lane < kMergeThreads / 32) s_warp[lane] = w;
        }
        __syncthreads();
        if (keep) {
            const int pos = total + incl - 1 + (warp > 0 ? s_warp[warp - 1] : 0);
            s_key[pos] = ((uint64_t)desc_key(r) << 32) | (uint32_t)s;
        }
        total += s_warp[kMergeThreads / 32 - 1];
        __syncthreads();
    }
    const int m = total;
    int M = 1;
    while (M < m) M <<= 1;
    for (int i = m + threadIdx.x; i < M; i += kMergeThreads) s_key[i] = ~0ull;
    __syncthreads();

    // 2. bitonic sort, ascending in key_less
    for (int k = 2; k <= M; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < M; i += kMergeThreads) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t x = s_key[i], y = s_key[ixj];
                    const bool up = (i & k) == 0;
                    if (up ? key_less(y, x, th, P) : key_less(x, y, th, P)) {
                        s_key[i] = y;
                        s_key[ixj] = x;
                    }
                }
            }
            __syncthreads();
        }
    }

    // 3. greedy leader clustering, exactly the sequential rule, in rounds of 32 candidates (sorted
    //    order): (a) every warp compares the round's candidates (one per lane) with a strided share
    //    of the leaders that existed when the round began, and the smallest matching leader index
    //    per candidate is reduced in shared memory; (b) warp 0 then walks the round in order: a
    //    candidate with such a match joins it (an older leader is always the earliest), otherwise
    //    it is compared with the leaders founded earlier in this round (one per lane), joins the
    //    first, or founds a new leader.  Leader records overwrite key slots <= the current
    //    candidate, whose keys the round already copied.
    {
        int L = 0;
        for (int q0 = 0; q0 < m; q0 += 32) {
            const int nb = min(32, m - q0);
            if (warp == 0) {
                if (lane < nb) {
                    const int sidx = (int)(uint32_t)s_key[q0 + lane];
                    s_csid[lane] = sidx;
                    s_ct[lane * 3] = __ldg(th + (int64_t)sidx * P);
                    s_ct[lane * 3 + 1] = __ldg(th + (int64_t)sidx * P + 1);
                    s_ct[lane * 3 + 2] = (P == 3) ? __ldg(th + (int64_t)sidx * P + 2) : 0.f;
                }
                s_cmin[lane] = 0x7fffffff;
            }
            __syncthreads();
            const int L0 = L;  // leaders founded before this round (uniform)
            if (lane < nb && L0 > 0) {
                const double t0 = s_ct[lane * 3], t1 = s_ct[lane * 3 + 1], t2 = s_ct[lane * 3 + 2];
                for (int l = warp; l < L0; l += kMergeThreads / 32) {
                    float l0, l1, l2 = 0.f;
                    if (l < kLeaderCache) {
                        l0 = s_lt[l * 3];
                        l1 = s_lt[l * 3 + 1];
                        l2 = s_lt[l * 3 + 2];
                    } else {
                        const int ls = (int)(uint32_t)s_key[l];
                        l0 = __ldg(th + (int64_t)ls * P);
                        l1 = __ldg(th + (int64_t)ls * P + 1);
                        if (P == 3) l2 = __ldg(th + (int64_t)ls * P + 2);
                    }
                    if (fabs(t0 - (double)l0) <= r0 && fabs(t1 - (double)l1) <= r1 &&
                        (P != 3 || fabs(t2 - (double)l2) <= r2)) {
                        atomicMin(&s_cmin[lane], l);  // first match of this warp's share = its smallest
                        break;
                    }
                }
            }
            __syncthreads();
            if (warp == 0) {
                for (int j = 0; j < nb; ++j) {
                    int found = s_cmin[j];
                    if (found == 0x7fffffff) {
                        found = -1;
                        const int nn = L - L0;  // leaders founded earlier in this round (< 32)
                        bool in = false;
                        if (lane < nn) {
                            const int l = L0 + lane;
                            float l0, l1, l2 = 0.f;
                            if (l < kLeaderCache) {
                                l0 = s_lt[l * 3];
                                l1 = s_lt[l * 3 + 1];
                                l2 = s_lt[l * 3 + 2];
                            } else {
                                const int ls = (int)(uint32_t)s_key[l];
                                l0 = __ldg(th + (int64_t)ls * P);
                                l1 = __ldg(th + (int64_t)ls * P + 1);
                                if (P == 3) l2 = __ldg(th + (int64_t)ls * P + 2);
                            }
                            in = fabs((double)s_ct[j * 3] - (double)l0) <= r0 &&
                                 fabs((double)s_ct[j * 3 + 1] - (double)l1) <= r1 &&
                                 (P != 3 || fabs((double)s_ct[j * 3 + 2] - (double)l2) <= r2);
                        }
                        const unsigned bal = __ballot_sync(0xffffffffu, in);
                        if (bal) found = L0 + __ffs(bal) - 1;
                    }
                    if (lane == 0) {
                        if (found >= 0) {
                            s_key[found] += (1ull << 32);
                        } else {
                            s_key[L] = (1ull << 32) | (uint32_t)s_csid[j];
                            if (L < kLeaderCache) {
                                s_lt[L * 3] = s_ct[j * 3];
                                s_lt[L * 3 + 1] = s_ct[j * 3 + 1];
                                s_lt[L * 3 + 2] = s_ct[j * 3 + 2];
                            }
                        }
                    }
                    if (found < 0) ++L;
                    __syncwarp();
                }
                if (lane == 0) s_m = L;
            }
            __syncthreads();
            L = s_m;  // every thread learns the round's leader count
        }
        if (m == 0 && threadIdx.x == 0) s_m = 0;
    }
    __syncthreads();

    // 4. emit leaders in creation order
    const int L = s_m;
    for (int l = threadIdx.x; l < L && l < a.capacity; l += kMergeThreads) {
        const uint64_t rec = s_key[l];
        const int sidx = (int)(uint32_t)rec;
        const int64_t o = (int64_t)e * a.capacity + l;
        for (int i = 0; i < P; ++i) a.t_theta[o * P + i] = __ldg(th + (int64_t)sidx * P + i);
        a.t_R[o] = __ldg(rr + sidx);
        a.t_seed[o] = sidx;
        a.t_size[o] = (int32_t)(rec >> 32);
    }
    if (threadIdx.x == 0) a.t_count[e] = L;
}

cudaError_t launch_merge(const MergeArgs &a0, int n_events, cudaStream_t stream) {
    if (n_events == 0) return cudaSuccess;
    int M = 1;
    while (M < a0.n_seeds) M <<= 1;
    const size_t smem = (size_t)M * sizeof(uint64_t);
    cudaError_t err = ensure_dynamic_smem(merge_kernel, smem);
    if (err != cudaSuccess) return err;
    MergeArgs a = a0;
    a.e_base = 0;
    merge_kernel<<<n_events, kMergeThreads, smem, stream>>>(a);
    return cudaGetLastError();
}

}  // namespace retina
