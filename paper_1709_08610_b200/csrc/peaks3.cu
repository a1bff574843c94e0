// peaks3.cu -- K2+K3 for P = 3 (the 3 x 3 x 3 neighbourhood of step (iii); reading
// Z6: strict local maxima over the EXISTING 26 neighbours with R >= R0), the workspace path of
// retina_find_peaks_ws.
//
// Pass 1 (peaks3_brick_kernel): grid (column blocks, events).  With the layout R[i][j][l] (l
// fastest), CTA (jb, e) owns the cells (i, j, l) of its TJ rows j in [jb TJ, jb TJ + TJ), for ALL i
// and l (TJ n2 = 2048 cells per plane for cfg4's 256^3), and walks i = 0 .. n0 - 1.  The block of
// plane i it needs -- rows j0 - 1 .. j0 + TJ (one halo row each side), all l -- is ONE contiguous
// range of the grid, so a producer warp streams each plane by a single TMA bulk copy
// (cp.async.bulk, mbarrier complete_tx) into a ring of kRing shared-memory slots; every cell is
// read from HBM once (the halo rows are the neighbouring CTAs' rows, read at about the same
// time: L2).  The consumer warps never meet at a block barrier: a slot is refilled once every
// consumer warp has arrived on its "empty" mbarrier.
// Consumers: per plane each thread loads its 4-cell groups (one 16-byte shared load each) and
// tests the threshold only; a group with some cell >= R0 (~8 % on cfg4) goes to the warp's queue.
// The queue is checked 32 groups at a time, one per lane (or after kDefer planes): the
// l-neighbours first, then, for a cell that beats them, its other 24 neighbours (max of 8 rows of
// 3, branch-free).  A plane is handed back to the producer only once no queued group needs it.
// A peak takes its place in its plane segment's list (plane i, column block jb: a contiguous
// range of linear indices) by a shared-memory atomic; each segment stores its TRUE count and its
// first kSegList peaks.  Measured on cfg4 (256^3 fp32 grids, B200): 0.44 of HBM per event grid
// (pure streaming through the same ring: 1.0), from 0.11 for the per-cell global-load scan.
//
// Pass 2 (peaks3_chunk_sum_kernel + peaks3_gather_kernel, one CTA per chunk of 512 segments and
// event): exclusive scan of the segment counts in segment order (= ascending linear index; a
// chunk's offset is the sum of the earlier chunks' totals), each segment's list sorted and copied
// to its offset (up to `capacity`), and, for a segment with more than kSegList peaks, a rescan of
// its cells with the same rule.  Integer sums in a fixed order: bit-deterministic, identical to the
// single-CTA path (T3).
#include "common.cuh"
#include "kernels.cuh"

namespace retina {

constexpr int kB3Threads = 512;  // gather / rescan CTAs
#ifndef RETINA_P3_THREADS
#define RETINA_P3_THREADS 256
#endif
constexpr int kCThreads = RETINA_P3_THREADS;  // consumer threads of a brick CTA (+ 1 producer warp)
#ifndef RETINA_P3_DEFER
#define RETINA_P3_DEFER 2   // planes a queued group may wait in its warp's queue
#endif
#ifndef RETINA_P3_RING
#define RETINA_P3_RING (RETINA_P3_DEFER + 4)
#endif
#ifndef RETINA_P3_CELLS
#define RETINA_P3_CELLS 2048
#endif
constexpr int kDefer = RETINA_P3_DEFER;
constexpr int kRing = RETINA_P3_RING;  // plane slots: i - 1, i, i + 1 resident, the rest in flight
constexpr int kSegList = 32;      // peaks a segment keeps from pass 1 (more: pass 2 rescans it)
#ifndef RETINA_P3_QUEUE
#define RETINA_P3_QUEUE 64
#endif
constexpr int kBlockCells = RETINA_P3_CELLS;  // cells of one plane block (TJ rows x n2)
constexpr int kGroups = (kBlockCells + 4 * RETINA_P3_THREADS - 1) / (4 * RETINA_P3_THREADS);  // 4-cell groups per thread
static_assert(kGroups >= 1 && kGroups <= 16, "4-cell groups per consumer thread");
// 4-cell groups a warp queues for the neighbour tests: at least one plane's worth (32 kGroups)
constexpr int kQueue = RETINA_P3_QUEUE > 32 * kGroups ? RETINA_P3_QUEUE : 32 * kGroups;

constexpr int kMaxSlotFloats = 10240;  // 40 KB per ring slot at most (kRing slots <= 200 KB)

// rows per column block for a given row length (n2 % 4 == 0, n2 <= 2048)
__host__ __device__ inline int b3_rows(int n1, int n2) {
    int tj = kBlockCells / n2;
    if (tj < 1) tj = 1;
    if (tj > n1) tj = n1;
    return tj;
}

bool peaks3_brick_ok(int n0, int n1, int n2) {
    if (n2 % 4 != 0 || n2 > 2048 || n0 > 8192) return false;
    const int tj = b3_rows(n1, n2);
    return (size_t)(tj + 2) * n2 <= (size_t)kMaxSlotFloats;
}

// pass 2 works on chunks of kB3Threads consecutive segments (one CTA each)
__host__ __device__ inline long long b3_chunks(long long nseg) { return (nseg + kB3Threads - 1) / kB3Threads; }

size_t peaks3_workspace_bytes(long long n_events, int n0, int n1, int n2) {
    const int tj = b3_rows(n1, n2);
    const long long nseg = (long long)n0 * ((n1 + tj - 1) / tj);
    // count, offset, then per segment kSegList indices and values; per chunk its peak total
    return (size_t)(n_events * nseg) * (2 * sizeof(int32_t) + (size_t)kSegList * (sizeof(int32_t) + sizeof(float))) +
           (size_t)(n_events * b3_chunks(nseg)) * sizeof(int32_t);
}

struct SegWs {
    int32_t *count, *offset, *idx;
    float *val;
    int32_t *ctot;  // [events][chunks]
    __device__ __forceinline__ static SegWs at(int32_t *ws, long long n_ev, long long nseg) {
        SegWs w;
        const long long n = n_ev * nseg;
        w.count = ws;
        w.offset = ws + n;
        w.idx = ws + 2 * n;
        w.val = reinterpret_cast<float *>(ws + 2 * n + n * kSegList);
        w.ctot = ws + 2 * n + 2 * n * kSegList;
        return w;
    }
};

__device__ __forceinline__ int b3_warp_incl_scan(int v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Block-wide ordered compaction of one group of flags (4 cells per thread, ascending with the
// thread index): writes the set cells' indices/values at list positions pos0 + rank (< lim).
// Returns the group's total.  Contains two __syncthreads.
__device__ __forceinline__ int b3_compact(unsigned mask, int cell0, const float4 v, int pos0, int lim,
                                          int32_t *oi, float *ov, int *s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cnt = __popc(mask);
    const int incl = b3_warp_incl_scan(cnt);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = (lane < kB3Threads / 32) ? s_warp[lane] : 0;
        w = b3_warp_incl_scan(w);
        if (lane < kB3Threads / 32) s_warp[lane] = w;
    }
    __syncthreads();
    int pos = pos0 + incl - cnt + (warp > 0 ? s_warp[warp - 1] : 0);
    const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        if (mask & (1u << c)) {
            if (pos < lim) {
                oi[pos] = cell0 + c;
                ov[pos] = vv[c];
            }
            ++pos;
        }
    }
    const int total = s_warp[kB3Threads / 32 - 1];
    return total;
}

// One producer warp (TMA loads) + kB3Threads / 32 consumer warps; the consumers never meet at a
// block barrier inside the plane loop: a plane slot is refilled once every consumer warp has
// arrived on the slot's "empty" mbarrier, and peaks take their position in the segment list by
// a shared-memory atomic (pass 2 sorts each list, so the output is still ascending and
// deterministic).
__global__ void __launch_bounds__(kCThreads + 32) peaks3_brick_kernel(PeakArgs a, int TJ, int32_t *ws) {
    extern __shared__ __align__(16) float4 s_ring4[];
    __shared__ __align__(8) uint64_t s_full[kRing], s_empty[kRing];
    float *ring = reinterpret_cast<float *>(s_ring4);
    int2 *s_queue = reinterpret_cast<int2 *>(ring + kRing * (TJ + 2) * a.n2);  // [warps][kQueue] candidates
    int *s_qn = reinterpret_cast<int *>(s_queue + (kCThreads / 32) * kQueue);    // [warps] queue fill
    int *s_cnt = s_qn + kCThreads / 32;                                           // [n0] per-plane peak counts
    const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
    const int NJB = gridDim.x, jb = blockIdx.x;
    const int e = a.e_base + blockIdx.y;
    const int j0 = jb * TJ, j1 = min(n1, j0 + TJ);
    const int rlo = max(0, j0 - 1), rhi = min(n1, j1 + 1);  // rows loaded: [rlo, rhi)
    const int slot = (TJ + 2) * n2;                          // floats per ring slot
    const int srow0 = rlo - (j0 - 1);                        // slot row of grid row rlo (0 or 1)
    const int64_t cells = (int64_t)n0 * n1 * n2;
    const float *g = a.R + (int64_t)e * cells;
    const long long nseg = (long long)n0 * NJB;
    const SegWs w = SegWs::at(ws, gridDim.y, nseg);
    const int64_t seg_base = (int64_t)blockIdx.y * nseg;
    const int Q = (j1 - j0) * n2;  // cells of this block per plane
    constexpr int kCons = kCThreads / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    for (int i = threadIdx.x; i < n0; i += blockDim.x) s_cnt[i] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&s_full[s], 1);
            mbar_init(&s_empty[s], kCons);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kCons) {  // producer warp: one lane streams the planes into the ring
        if (lane == 0) {
            const uint32_t bytes = (uint32_t)(rhi - rlo) * n2 * 4u;
            for (int p = 0; p < n0; ++p) {
                const int s = p % kRing;
                if (p >= kRing) mbar_wait(&s_empty[s], (uint32_t)(((p - kRing) / kRing) & 1));
                fence_proxy_async();
                mbar_arrive_expect_tx(&s_full[s], bytes);
                bulk_g2s(ring + s * slot + srow0 * n2, g + ((int64_t)p * n1 + rlo) * n2, bytes, &s_full[s]);
            }
        }
    } else {
        const float NEG = __int_as_float(0xff800000);  // -inf: a missing neighbour
        const float thr = a.threshold;
        // this thread's two 4-cell groups of every plane block (fixed over the planes): position and
        // shared-memory offset inside a ring slot
        int gjj[kGroups], gl[kGroups], goff[kGroups];
        bool gok[kGroups];
#pragma unroll
        for (int gi = 0; gi < kGroups; ++gi) {
            const int q = (gi * kCThreads + threadIdx.x) * 4;
            gok[gi] = q < Q;
            gjj[gi] = q / n2;
            gl[gi] = q - gjj[gi] * n2;
            goff[gi] = (gjj[gi] + 1) * n2 + gl[gi];
        }
        // this warp's queue of candidates (plane, packed (row, column)), checked 32 at a time; a
        // candidate of plane p needs planes p - 1 .. p + 1, so a plane is released (its slot may be
        // refilled) only once no queued candidate needs it
        int2 *queue = s_queue + warp * kQueue;
        int nq = 0, q0 = 0;   // queued entries, plane of the oldest
        int released = -1;    // planes <= released are handed back to the producer
        auto check = [&](int2 ent) {  // strict test of one candidate against its other 24 neighbours
            const int i = ent.x, jj = ent.y >> 16, lc = ent.y & 0xffff;
            RETINA_ASSERT(i >= 0 && i < n0 && jj >= 0 && jj < j1 - j0 && lc >= 0 && lc < n2);
            const int r = jj + 1, jg = j0 + jj;
            const float *pc = ring + (i % kRing) * slot;
            const float *pm = (i > 0) ? ring + ((i - 1) % kRing) * slot : pc;  // pc: a dummy, masked
            const float *pp = (i + 1 < n0) ? ring + ((i + 1) % kRing) * slot : pc;
            const float x = pc[r * n2 + lc];
            const int la = max(lc - 1, 0), lb = min(lc + 1, n2 - 1);
            const bool hasl = lc > 0, hasr = lc + 1 < n2;
            const bool up = jg > 0, down = jg + 1 < n1, hm = i > 0, hp = i + 1 < n0;
            auto rowmax = [&](const float *p, int rr, bool ok) {
                const float *q = p + rr * n2;
                const float m3 = fmaxf(fmaxf(hasl ? q[la] : NEG, q[lc]), hasr ? q[lb] : NEG);
                return ok ? m3 : NEG;
            };
            float mx = fmaxf(rowmax(pc, r - 1, up), rowmax(pc, r + 1, down));
            mx = fmaxf(mx, fmaxf(rowmax(pm, r - 1, hm && up), rowmax(pm, r, hm)));
            mx = fmaxf(mx, fmaxf(rowmax(pm, r + 1, hm && down), rowmax(pp, r - 1, hp && up)));
            mx = fmaxf(mx, fmaxf(rowmax(pp, r, hp), rowmax(pp, r + 1, hp && down)));
            if (x > mx) {
                const int64_t seg = seg_base + (int64_t)i * NJB + jb;
                const int p = atomicAdd(&s_cnt[i], 1);
                if (p < kSegList) {
                    w.idx[seg * kSegList + p] = (int)(((int64_t)i * n1 + j0 + jj) * n2) + lc;
                    w.val[seg * kSegList + p] = x;
                }
            }
        };
        auto group = [&](int2 ent) {  // a queued 4-cell group: l-neighbour test, then check()
            const int i = ent.x, jj = ent.y >> 16, l = ent.y & 0xffff;
            const float *row = ring + (i % kRing) * slot + (jj + 1) * n2;
            const float4 v4 = *reinterpret_cast<const float4 *>(row + l);
            const float lf = (l > 0) ? row[l - 1] : NEG;
            const float rt = (l + 4 < n2) ? row[l + 4] : NEG;
            const unsigned k = ((v4.x >= thr) & (v4.x > lf) & (v4.x > v4.y)) |
                               (((v4.y >= thr) & (v4.y > v4.x) & (v4.y > v4.z)) << 1) |
                               (((v4.z >= thr) & (v4.z > v4.y) & (v4.z > v4.w)) << 2) |
                               (((v4.w >= thr) & (v4.w > v4.z) & (v4.w > rt)) << 3);
            for (unsigned m = k; m; m &= m - 1) check(make_int2(i, ent.y + (__ffs(m) - 1)));
        };
        auto flush = [&]() {
            __syncwarp();
            for (int base = 0; base < nq; base += 32)
                if (base + lane < nq) group(queue[base + lane]);
            __syncwarp();
            nq = 0;
        };
        mbar_wait(&s_full[0], 0u);
        for (int i = 0; i < n0; ++i) {
            if (i + 1 < n0) mbar_wait(&s_full[(i + 1) % kRing], (uint32_t)(((i + 1) / kRing) & 1));
            const float *pc = ring + (i % kRing) * slot;
            // stage 1 (every cell, uniform work): one 16-byte load and the threshold per 4 cells; the
            // groups with some cell >= R0 (~8 % for cfg4) are queued for the neighbour tests
            unsigned grp = 0u;
#pragma unroll
            for (int gi = 0; gi < kGroups; ++gi) {
#ifdef RETINA_P3_NOCOMPUTE
                continue;
#endif
                if (!gok[gi]) continue;
                const float4 v4 = *reinterpret_cast<const float4 *>(pc + goff[gi]);
                if (fmaxf(fmaxf(v4.x, v4.y), fmaxf(v4.z, v4.w)) >= thr) grp |= 1u << gi;
            }
            const int nc = __popc(grp);
            const unsigned who = __ballot_sync(0xffffffffu, nc != 0);
            if (who) {
                const int total = __reduce_add_sync(0xffffffffu, nc);  // <= 32 kGroups <= kQueue
                if (nq + total > kQueue) flush();
                if (nq == 0) q0 = i;
                // positions by a shared counter: the order inside the queue does not matter
                if (lane == 0) s_qn[warp] = nq;
                __syncwarp();
                int pos = nc ? atomicAdd(&s_qn[warp], nc) : 0;
                for (unsigned m = grp; m; m &= m - 1) {
                    const int gi = __ffs(m) - 1;
                    queue[pos++] = make_int2(i, (gjj[gi] << 16) | gl[gi]);
                }
                nq += total;
            }
            // check the queue when it fills a round, or before its oldest plane would hold the ring
            // back, or at the end
            if (nq >= 32 || (nq > 0 && i - q0 >= kDefer - 1) || i + 1 == n0) flush();
            // hand back every plane no queued candidate (of planes >= q0) and no later plane needs
            const int rel_to = (nq == 0) ? i - 1 : min(i - 1, q0 - 2);
            __syncwarp();
            if (lane == 0)
                for (int p = released + 1; p <= rel_to; ++p) mbar_arrive(&s_empty[p % kRing]);
            released = max(released, rel_to);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n0; i += blockDim.x) w.count[seg_base + (int64_t)i * NJB + jb] = s_cnt[i];
}

// Ordered scan of cells [c_begin, c_end) of one event with the plain global-memory rule (pass 2's
// rescan of a segment with more than kSegList peaks); writes at pos0 + rank (< cap).
__device__ int b3_rescan(const PeakArgs &a, const float *g, int32_t *oi, float *ov, int c_begin, int c_end,
                         int pos0, int *s_warp) {
    const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
    int total = 0;
    for (int base = c_begin; base < c_end; base += kB3Threads) {
        const int c = base + threadIdx.x;
        bool pk = false;
        if (c < c_end) {
            const float v = g[c];
            if (v >= a.threshold) {
                const int l = c % n2, t = c / n2, j = t % n1, i = t / n1;
                pk = true;
                for (int di = -1; di <= 1 && pk; ++di)
                    for (int dj = -1; dj <= 1 && pk; ++dj)
                        for (int dl = -1; dl <= 1 && pk; ++dl) {
                            const int ii = i + di, jj = j + dj, ll = l + dl;
                            if ((di | dj | dl) == 0 || ii < 0 || ii >= n0 || jj < 0 || jj >= n1 || ll < 0 || ll >= n2)
                                continue;
                            if (!(v > g[((int64_t)ii * n1 + jj) * n2 + ll])) pk = false;
                        }
            }
        }
        const float4 vv = make_float4(pk ? g[c] : 0.f, 0.f, 0.f, 0.f);
        total += b3_compact(pk ? 1u : 0u, c, vv, pos0 + total, a.capacity, oi, ov, s_warp);
        __syncthreads();
    }
    return total;
}

__device__ __forceinline__ int b3_block_sum(int v, int *s_warp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) s_warp[warp] = v;
    __syncthreads();
    int t = 0;
    for (int k = 0; k < kB3Threads / 32; ++k) t += s_warp[k];
    return t;
}

// pass 2a: the peak total of every chunk of kB3Threads segments (grid (chunks, events))
__global__ void __launch_bounds__(kB3Threads) peaks3_chunk_sum_kernel(PeakArgs a, int NJB, int32_t *ws) {
    __shared__ int s_warp[kB3Threads / 32];
    const long long nseg = (long long)a.n0 * NJB, nch = b3_chunks(nseg);
    const SegWs w = SegWs::at(ws, gridDim.y, nseg);
    const long long s = (long long)blockIdx.x * kB3Threads + threadIdx.x;
    const int n = (s < nseg) ? w.count[(int64_t)blockIdx.y * nseg + s] : 0;
    const int t = b3_block_sum(n, s_warp);
    if (threadIdx.x == 0) w.ctot[(int64_t)blockIdx.y * nch + blockIdx.x] = t;
}

// pass 2b (grid (chunks, events)): the chunk's offset is the sum of the earlier chunks' totals;
// a block scan places its segments, whose lists are sorted and copied; a segment with more than
// kSegList peaks is rescanned in place; the last chunk writes the event's true count
__global__ void __launch_bounds__(kB3Threads) peaks3_gather_kernel(PeakArgs a, int NJB, const int32_t *ws) {
    __shared__ int s_warp[kB3Threads / 32];
    const int e = a.e_base + blockIdx.y, c = blockIdx.x;
    const long long nseg = (long long)a.n0 * NJB, nch = b3_chunks(nseg);
    const SegWs w = SegWs::at(const_cast<int32_t *>(ws), gridDim.y, nseg);
    const int64_t sb = (int64_t)blockIdx.y * nseg;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t *oi = a.idx + (int64_t)e * a.capacity;
    float *ov = a.val + (int64_t)e * a.capacity;
    int pre = 0;
    for (long long k = threadIdx.x; k < c; k += kB3Threads) pre += w.ctot[(int64_t)blockIdx.y * nch + k];
    const int prefix = b3_block_sum(pre, s_warp);
    __syncthreads();
    const long long s = (long long)c * kB3Threads + threadIdx.x;
    const int n = (s < nseg) ? w.count[sb + s] : 0;
    const int incl = b3_warp_incl_scan(n);
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int x = (lane < kB3Threads / 32) ? s_warp[lane] : 0;
        x = b3_warp_incl_scan(x);
        if (lane < kB3Threads / 32) s_warp[lane] = x;
    }
    __syncthreads();
    const int off = prefix + incl - n + (warp > 0 ? s_warp[warp - 1] : 0);
    const int chunk_total = s_warp[kB3Threads / 32 - 1];
    if (c == nch - 1 && threadIdx.x == 0) a.cnt[e] = prefix + chunk_total;
    bool overflow = false;
    if (s < nseg) {
        w.offset[sb + s] = off;
        if (n > kSegList) {
            overflow = true;
        } else if (n > 0 && off < a.capacity) {
            // pass 1 stored the segment's peaks in arrival order: sort by index (<= kSegList)
            int ki[kSegList];
            float kv[kSegList];
#pragma unroll
            for (int k = 0; k < kSegList; ++k) {
                if (k < n) {
                    ki[k] = w.idx[(sb + s) * kSegList + k];
                    kv[k] = w.val[(sb + s) * kSegList + k];
                }
            }
            for (int k = 0; k < n && off + k < a.capacity; ++k) {  // selection of the k-th smallest
                int best = k;
                for (int m = k + 1; m < n; ++m)
                    if (ki[m] < ki[best]) best = m;
                const int ti = ki[best];
                const float tv = kv[best];
                ki[best] = ki[k];
                kv[best] = kv[k];
                oi[off + k] = ti;
                ov[off + k] = tv;
            }
        }
    }
    // this chunk's segments with more than kSegList peaks, in order, rescanned by the whole block
    const unsigned bal = __ballot_sync(0xffffffffu, overflow);
    __shared__ int s_list[kB3Threads];
    __shared__ int s_nlist;
    if (!__syncthreads_or(overflow)) return;
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int k = 0; k < kB3Threads / 32; ++k) {
            const int cc = s_warp[k];
            s_warp[k] = acc;
            acc += cc;
        }
        s_nlist = acc;
    }
    __syncthreads();
    if (overflow) s_list[s_warp[warp] + __popc(bal & ((1u << lane) - 1u))] = (int)threadIdx.x;
    __syncthreads();
    const int nl = s_nlist;
    const int tj = b3_rows(a.n1, a.n2);
    const float *g = a.R + (int64_t)e * a.n0 * a.n1 * a.n2;
    for (int k = 0; k < nl; ++k) {
        const long long sg = (long long)c * kB3Threads + s_list[k];
        const int pos0 = w.offset[sb + sg];
        if (pos0 >= a.capacity) break;  // uniform: later segments start further on
        const int i = (int)(sg / NJB), jb = (int)(sg - (long long)i * NJB);
        const int j0 = jb * tj, j1 = min(a.n1, j0 + tj);
        const int c0 = (int)(((int64_t)i * a.n1 + j0) * a.n2), c1 = (int)(((int64_t)i * a.n1 + j1) * a.n2);
        b3_rescan(a, g, oi, ov, c0, c1, pos0, s_warp);
    }
}

cudaError_t launch_find_peaks3_brick(const PeakArgs &a0, int n_events, int32_t *ws, cudaStream_t stream) {
    const int TJ = b3_rows(a0.n1, a0.n2);
    const int NJB = (a0.n1 + TJ - 1) / TJ;
    const size_t smem = (size_t)kRing * (TJ + 2) * a0.n2 * sizeof(float) +
                        (size_t)(kCThreads / 32) * kQueue * sizeof(int2) +
                        ((size_t)kCThreads / 32 + a0.n0) * sizeof(int);
    cudaError_t err = ensure_dynamic_smem(peaks3_brick_kernel, smem);
    if (err != cudaSuccess) return err;
    for (int e0 = 0; e0 < n_events; e0 += 65535) {
        PeakArgs a = a0;
        a.e_base = e0;
        const int ne = min(65535, n_events - e0);
        // this launch's workspace: ne events from the start of the caller's buffer (the launches
        // run in stream order, so each reuses it)
        peaks3_brick_kernel<<<dim3(NJB, ne), kCThreads + 32, smem, stream>>>(a, TJ, ws);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        const unsigned nch = (unsigned)b3_chunks((long long)a0.n0 * NJB);
        peaks3_chunk_sum_kernel<<<dim3(nch, ne), kB3Threads, 0, stream>>>(a, NJB, ws);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
        peaks3_gather_kernel<<<dim3(nch, ne), kB3Threads, 0, stream>>>(a, NJB, ws);
        err = cudaGetLastError();
        if (err != cudaSuccess) return err;
    }
    return cudaSuccess;
}

}  // namespace retina
