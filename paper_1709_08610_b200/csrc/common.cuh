// common.cuh -- device helpers shared by the retina kernels (sm_100a only).
//
// * ex2.approx.ftz.f32 (one MUFU.EX2): exp(-s^2/sigma^2) = 2^(-K s^2), K = log2(e)/sigma^2.
// * TMA bulk copies (cp.async.bulk, SASS UBLKCP) of an event's hits into shared memory,
//   completed on an mbarrier (complete_tx), through the HitStage helper below.
// * Exact-difference helpers (TwoSum / TwoProd) for residuals whose plain fp32
//   difference would lose the 1e-5 parity budget.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Bounds checks of the index arithmetic for a debug build (-DRETINA_DEBUG: device-side asserts;
// compute-sanitizer is not available on this pool); compiled out otherwise.
#ifdef RETINA_DEBUG
#include <cassert>
#define RETINA_ASSERT(cond) assert(cond)
#else
#define RETINA_ASSERT(cond) ((void)0)
#endif

#include <map>
#include <mutex>
#include <utility>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "retina kernels target sm_100a only"
#endif

namespace retina {

constexpr int kMaxStageHits = 12288;  // 192 KiB of float4 hits per CTA at most

// Raises a kernel's dynamic shared-memory limit once per (device, kernel, size): the only state
// the library keeps is this attribute cache, keyed by the kernel's address.  Skipping the call
// when the limit is already high enough keeps launches free of non-stream API calls, so a
// sequence of retina calls can be captured into a CUDA graph.
inline cudaError_t ensure_dynamic_smem_impl(const void *kern, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void *>, int> granted;
    int dev = 0;
    cudaError_t err = cudaGetDevice(&dev);
    if (err != cudaSuccess) return err;
    std::lock_guard<std::mutex> lock(mu);
    auto it = granted.find({dev, kern});
    if (it != granted.end() && (int)bytes <= it->second) return cudaSuccess;
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (err == cudaSuccess) granted[{dev, kern}] = (int)bytes;
    return err;
}

template <class Kernel>
inline cudaError_t ensure_dynamic_smem(Kernel kern, size_t bytes) {
    return ensure_dynamic_smem_impl(reinterpret_cast<const void *>(kern), bytes);
}

__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Knuth TwoSum: hi + lo == a + b exactly (round-to-nearest fp32, no FTZ issues for
// the magnitudes used here: mm coordinates).
__device__ __forceinline__ void two_sum(float a, float b, float &hi, float &lo) {
    float s = __fadd_rn(a, b);
    float bb = __fsub_rn(s, a);
    lo = __fadd_rn(__fsub_rn(a, __fsub_rn(s, bb)), __fsub_rn(b, bb));
    hi = s;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!done);
}

// One bulk global->shared copy (bytes % 16 == 0, both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Stages one event's hits through shared memory with TMA bulk copies.
//
// `cap` float4 slots of dynamic shared memory.  If the event fits (n <= cap) the hits are
// loaded once and stay RESIDENT for every pass (multi-start re-reads them n_iters+1 times).
// Otherwise they STREAM in chunks of cap/2 through a double buffer: the copy of chunk c+1
// is in flight while chunk c is consumed.  Every thread of the CTA must call pass() the
// same number of times (it contains __syncthreads()).
struct HitStage {
    float4 *buf;        // dynamic smem, cap float4
    uint64_t *bar;      // 2 mbarriers in static smem
    const float4 *g;    // this event's hits in global memory
    int n;              // hits in this event
    int cap;            // float4 slots
    uint32_t loads;     // bulk loads issued so far (uniform across the CTA)
    bool resident;

    __device__ __forceinline__ void init(float4 *sbuf, uint64_t *sbar, const float4 *ghits, int nhits,
                                         int capacity) {
        buf = sbuf;
        bar = sbar;
        g = ghits;
        n = nhits;
        cap = capacity;
        loads = 0;
        resident = false;
        if (threadIdx.x == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            fence_mbar_init();
        }
        __syncthreads();
    }

    __device__ __forceinline__ void issue(int start, int len, int slot) {
        // slot 0 = first half (or whole buffer when resident), slot 1 = second half
        const uint32_t bytes = static_cast<uint32_t>(len) * 16u;
        fence_proxy_async();
        mbar_arrive_expect_tx(&bar[slot], bytes);
        bulk_g2s(buf + (slot ? cap / 2 : 0), g + start, bytes, &bar[slot]);
    }

    // Resident mode only: brings the event's hits into shared memory now (every thread waits), so
    // the caller can index them before the first pass.  Returns whether they are resident.
    __device__ __forceinline__ bool load_resident() {
        if (n <= 0 || n > cap) return false;
        if (!resident) {
            if (threadIdx.x == 0) issue(0, n, 0);
            mbar_wait(&bar[0], 0u);
            resident = true;
        }
        return true;
    }

    // Calls body(const float4* hits, int count) for consecutive chunks covering all hits.
    template <class F>
    __device__ __forceinline__ void pass(F &&body) {
        if (n <= 0) return;
        if (n <= cap) {
            if (!resident) {  // n is fixed per CTA, so a CTA is resident or streaming for life
                if (threadIdx.x == 0) issue(0, n, 0);
                mbar_wait(&bar[0], 0u);
                resident = true;
            }
            body(static_cast<const float4 *>(buf), n);
            return;
        }
        const int ch = cap / 2;
        const int nch = (n + ch - 1) / ch;
        // chunk c uses slot (loads + c) & 1 and waits parity ((loads + c) >> 1) & 1
        if (threadIdx.x == 0) issue(0, min(ch, n), loads & 1u);
        for (int c = 0; c < nch; ++c) {
            const uint32_t k = loads + c;
            if (c + 1 < nch && threadIdx.x == 0) {
                const int s = (c + 1) * ch;
                issue(s, min(ch, n - s), (k + 1) & 1u);
            }
            mbar_wait(&bar[k & 1u], (k >> 1) & 1u);
            const int s = c * ch;
            body(static_cast<const float4 *>(buf + ((k & 1u) ? ch : 0)), min(ch, n - s));
            __syncthreads();
        }
        loads += nch;
    }
};

}  // namespace retina
