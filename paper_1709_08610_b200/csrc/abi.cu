// abi.cu -- the extern "C" boundary declared in include/retina.h: host-side validation,
// derived fp32 constants (rounded once from fp64), and launches on the caller's stream.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>

#include "../../include/retina.h"
#include "common.cuh"
#include "kernels.cuh"

namespace {

thread_local char g_last_error[512] = "";

int fail(int status, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
    return status;
}

int cuda_fail(cudaError_t err, const char *where) {
    return fail(RETINA_ECUDA, "%s: %s (%s)", where, cudaGetErrorString(err), cudaGetErrorName(err));
}

int model_P(int model) {
    return model == RETINA_SLOPE3 ? 3 : (model == RETINA_LINE2D || model == RETINA_SLOPE2) ? 2 : -1;
}

bool finite_pos(float v) { return std::isfinite(v) && v > 0.f; }

// -log2(e)/sigma^2 and 2/sigma^2 from the fp32 sigma, in fp64, rounded once.
float neg_k(float sigma) {
    const double s = sigma;
    return (float)(-1.4426950408889634074 / (s * s));
}
float c2_of(float sigma) {
    const double s = sigma;
    return (float)(2.0 / (s * s));
}
// sqrt(log2(e)) / sigma and (2 / sigma^2) / that, in fp64, rounded once (SLOPE3 multi-start)
float sk_of(float sigma) { return (float)(1.2011224087864498 / (double)sigma); }
float c2s_of(float sigma) { return (float)(2.0 / ((double)sigma * 1.2011224087864498)); }

int stage_cap(int32_t hint, int dflt) {
    if (hint <= 0) return dflt;
    int c = ((hint + 31) / 32) * 32;
    if (c < 64) c = 64;
    if (c > retina::kMaxStageHits) c = retina::kMaxStageHits;
    return c;
}

int check_events(const retina_events *ev) {
    if (!ev) return fail(RETINA_EINVAL, "ev is NULL");
    if (ev->n_events < 0) return fail(RETINA_EINVAL, "n_events < 0 (%d)", ev->n_events);
    if (ev->n_events > 0 && !ev->offsets) return fail(RETINA_EINVAL, "offsets is NULL");
    if (((uintptr_t)ev->hits & 15u) != 0) return fail(RETINA_EINVAL, "hits must be 16-byte aligned");
    if (!std::isfinite(ev->z_ref)) return fail(RETINA_EINVAL, "z_ref is not finite");
    if (ev->max_event_hits < 0) return fail(RETINA_EINVAL, "max_event_hits < 0");
    return RETINA_OK;
}

}  // namespace

extern "C" {

const char *retina_status_string(int status) {
    switch (status) {
        case RETINA_OK: return "RETINA_OK";
        case RETINA_EINVAL: return "RETINA_EINVAL: invalid argument";
        case RETINA_EUNSUPPORTED: return "RETINA_EUNSUPPORTED: size or option not supported";
        case RETINA_ECUDA: return "RETINA_ECUDA: CUDA launch or device error";
    }
    return "unknown retina status";
}

const char *retina_last_error(void) { return g_last_error; }

const char *retina_version(void) { return "retina-b200 0.1 sm_100a"; }

int retina_grid_response(const retina_events *ev, int model, float sigma, const int32_t *axis_len,
                         const float *const *axis_nodes, float *response, void *stream) {
    return retina_grid_response_ex(ev, model, sigma, axis_len, axis_nodes, response, RETINA_GRID_AUTO, stream);
}

// pairs every grid kernel but the culled one contracts: hits x cells, added on the device
__global__ void add_grid_pairs_kernel(const int32_t *offsets, int n_events, long long cells, unsigned long long *pairs) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd(pairs, (unsigned long long)(offsets[n_events] - offsets[0]) * (unsigned long long)cells);
}

int retina_grid_response_ex(const retina_events *ev, int model, float sigma, const int32_t *axis_len,
                            const float *const *axis_nodes, float *response, int algorithm, void *stream) {
    return retina_grid_response_ex2(ev, model, sigma, axis_len, axis_nodes, response, algorithm, nullptr, stream);
}

int retina_grid_response_ex2(const retina_events *ev, int model, float sigma, const int32_t *axis_len,
                             const float *const *axis_nodes, float *response, int algorithm,
                             unsigned long long *pairs_evaluated, void *stream) {
    g_last_error[0] = 0;
    int st = check_events(ev);
    if (st) return st;
    const int P = model_P(model);
    if (P < 0) return fail(RETINA_EINVAL, "unknown model %d", model);
    if (!finite_pos(sigma)) return fail(RETINA_EINVAL, "sigma must be finite and > 0");
    if (!axis_len || !axis_nodes) return fail(RETINA_EINVAL, "axis_len/axis_nodes is NULL");
    long long cells = 1;
    for (int i = 0; i < P; ++i) {
        if (axis_len[i] < 2) return fail(RETINA_EINVAL, "axis_len[%d] = %d < 2", i, axis_len[i]);
        if (!axis_nodes[i]) return fail(RETINA_EINVAL, "axis_nodes[%d] is NULL", i);
        cells *= axis_len[i];
    }
    if (cells > 0x7fffffffLL) return fail(RETINA_EUNSUPPORTED, "more than 2^31-1 cells per event");
    if (ev->n_events > 0 && !response) return fail(RETINA_EINVAL, "response is NULL");
    if (algorithm < RETINA_GRID_AUTO || algorithm > RETINA_GRID_TENSOR_F16_CULLED)
        return fail(RETINA_EINVAL, "unknown grid algorithm %d", algorithm);
    if (algorithm == RETINA_GRID_SEPARABLE && model == RETINA_LINE2D)
        return fail(RETINA_EUNSUPPORTED, "LINE2D residual does not factorise: no separable grid");
    if (algorithm >= RETINA_GRID_TENSOR && model == RETINA_LINE2D)
        return fail(RETINA_EUNSUPPORTED, "LINE2D residual does not factorise: no tensor-core grid");
    if (algorithm == RETINA_GRID_AUTO)
        algorithm = (model == RETINA_LINE2D)   ? RETINA_GRID_DIRECT
                                               : RETINA_GRID_TENSOR_F16;
    retina::GridArgs a{};
    a.offsets = ev->offsets;
    a.hits = reinterpret_cast<const float4 *>(ev->hits);
    a.z_ref = ev->z_ref;
    a.negK = neg_k(sigma);
    a.n0 = axis_len[0];
    a.n1 = axis_len[1];
    a.n2 = (P == 3) ? axis_len[2] : 1;
    a.nodes0 = axis_nodes[0];
    a.nodes1 = axis_nodes[1];
    a.nodes2 = (P == 3) ? axis_nodes[2] : nullptr;
    a.R = response;
    a.cap = stage_cap(ev->max_event_hits, 2048);
    a.pairs = (algorithm == RETINA_GRID_TENSOR_F16_CULLED) ? pairs_evaluated : nullptr;
    cudaError_t err;
    if (algorithm == RETINA_GRID_TENSOR)
        err = retina::launch_grid_tensor(model, a, ev->n_events, (cudaStream_t)stream);
    else if (algorithm == RETINA_GRID_TENSOR_F16 || algorithm == RETINA_GRID_TENSOR_F16_CULLED)
        err = retina::launch_grid_tensor16p(model, a, ev->n_events, (cudaStream_t)stream,
                                            algorithm == RETINA_GRID_TENSOR_F16_CULLED);
    else if (algorithm == RETINA_GRID_TENSOR_F16_PAIR)
        err = retina::launch_grid_tensor16x2(model, a, ev->n_events, (cudaStream_t)stream);
    else if (algorithm == RETINA_GRID_TENSOR_F16_SINGLE)
        err = retina::launch_grid_tensor16(model, a, ev->n_events, (cudaStream_t)stream);
    else if (algorithm == RETINA_GRID_SEPARABLE)
        err = retina::launch_grid_separable(model, a, ev->n_events, (cudaStream_t)stream);
    else
        err = retina::launch_grid_response(model, a, ev->n_events, (cudaStream_t)stream);
    if (err == cudaSuccess && pairs_evaluated && ev->n_events > 0 && !a.pairs) {
        add_grid_pairs_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ev->offsets, ev->n_events, cells, pairs_evaluated);
        err = cudaGetLastError();
    }
    if (err != cudaSuccess) return cuda_fail(err, "retina_grid_response");
    return RETINA_OK;
}

// The peak rule is symmetric in the axes, so the finder runs on the grid as a dense array in
// memory order: (n0, n1) for P = 2, (n2, n0, n1) for P = 3 (z0 planes outermost, Z37).
static void memory_dims(int P, const int32_t *axis_len, int &d0, int &d1, int &d2) {
    if (P == 3) {
        d0 = axis_len[2];
        d1 = axis_len[0];
        d2 = axis_len[1];
    } else {
        d0 = axis_len[0];
        d1 = axis_len[1];
        d2 = 1;
    }
}

int retina_find_peaks(const float *response, int32_t n_events, int32_t P, const int32_t *axis_len,
                      float threshold, int32_t capacity, int32_t *peak_index, float *peak_value,
                      int32_t *peak_count, void *stream) {
    g_last_error[0] = 0;
    if (n_events < 0) return fail(RETINA_EINVAL, "n_events < 0");
    if (P != 2 && P != 3) return fail(RETINA_EINVAL, "P must be 2 or 3 (got %d)", P);
    if (!axis_len) return fail(RETINA_EINVAL, "axis_len is NULL");
    if (capacity < 0) return fail(RETINA_EINVAL, "capacity < 0");
    if (std::isnan(threshold)) return fail(RETINA_EINVAL, "threshold is NaN");
    long long cells = 1;
    for (int i = 0; i < P; ++i) {
        if (axis_len[i] < 2) return fail(RETINA_EINVAL, "axis_len[%d] = %d < 2", i, axis_len[i]);
        cells *= axis_len[i];
    }
    if (cells > 0x7fffffffLL) return fail(RETINA_EUNSUPPORTED, "more than 2^31-1 cells per event");
    if (n_events == 0) return RETINA_OK;
    if (!response || !peak_count || (capacity > 0 && (!peak_index || !peak_value)))
        return fail(RETINA_EINVAL, "NULL device pointer");
    retina::PeakArgs a{};
    a.R = response;
    memory_dims(P, axis_len, a.n0, a.n1, a.n2);
    a.P = P;
    a.threshold = threshold;
    a.capacity = capacity;
    a.idx = peak_index;
    a.val = peak_value;
    a.cnt = peak_count;
    const cudaError_t err = retina::launch_find_peaks(a, n_events, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "retina_find_peaks");
    return RETINA_OK;
}

size_t retina_find_peaks_workspace_size(int32_t n_events, int32_t P, const int32_t *axis_len) {
    if (n_events <= 0 || (P != 2 && P != 3) || !axis_len) return 0;
    long long cells = 1;
    for (int i = 0; i < P; ++i) cells *= (axis_len[i] > 0 ? axis_len[i] : 0);
    if (cells <= 0 || cells > 0x7fffffffLL) return 0;
    int d0, d1, d2;
    memory_dims(P, axis_len, d0, d1, d2);
    return retina::peaks_workspace_bytes(n_events, P, d0, d1, d2);
}

int retina_find_peaks_ws(const float *response, int32_t n_events, int32_t P, const int32_t *axis_len,
                         float threshold, int32_t capacity, int32_t *peak_index, float *peak_value,
                         int32_t *peak_count, void *workspace, size_t workspace_bytes, void *stream) {
    g_last_error[0] = 0;
    if (n_events < 0) return fail(RETINA_EINVAL, "n_events < 0");
    if (P != 2 && P != 3) return fail(RETINA_EINVAL, "P must be 2 or 3 (got %d)", P);
    if (!axis_len) return fail(RETINA_EINVAL, "axis_len is NULL");
    if (capacity < 0) return fail(RETINA_EINVAL, "capacity < 0");
    if (std::isnan(threshold)) return fail(RETINA_EINVAL, "threshold is NaN");
    long long cells = 1;
    for (int i = 0; i < P; ++i) {
        if (axis_len[i] < 2) return fail(RETINA_EINVAL, "axis_len[%d] = %d < 2", i, axis_len[i]);
        cells *= axis_len[i];
    }
    if (cells > 0x7fffffffLL) return fail(RETINA_EUNSUPPORTED, "more than 2^31-1 cells per event");
    if (n_events == 0) return RETINA_OK;
    if (!response || !peak_count || (capacity > 0 && (!peak_index || !peak_value)))
        return fail(RETINA_EINVAL, "NULL device pointer");
    const size_t need = retina_find_peaks_workspace_size(n_events, P, axis_len);
    if (!workspace || workspace_bytes < need)
        return fail(RETINA_EINVAL, "workspace of %zu bytes needed (got %zu)", need, workspace_bytes);
    retina::PeakArgs a{};
    a.R = response;
    memory_dims(P, axis_len, a.n0, a.n1, a.n2);
    a.P = P;
    a.threshold = threshold;
    a.capacity = capacity;
    a.idx = peak_index;
    a.val = peak_value;
    a.cnt = peak_count;
    const cudaError_t err =
        retina::launch_find_peaks_ws(a, n_events, static_cast<int32_t *>(workspace), (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "retina_find_peaks_ws");
    return RETINA_OK;
}

int retina_estimate_peaks(const float *response, int32_t n_events, int32_t P, const int32_t *axis_len,
                          const float *const *axis_nodes, const int32_t *peak_index, const int32_t *peak_count,
                          int32_t capacity, float *peak_theta, void *stream) {
    g_last_error[0] = 0;
    if (n_events < 0) return fail(RETINA_EINVAL, "n_events < 0");
    if (P != 2 && P != 3) return fail(RETINA_EINVAL, "P must be 2 or 3 (got %d)", P);
    if (!axis_len || !axis_nodes) return fail(RETINA_EINVAL, "axis_len/axis_nodes is NULL");
    if (capacity < 0) return fail(RETINA_EINVAL, "capacity < 0");
    long long cells = 1;
    for (int i = 0; i < P; ++i) {
        if (axis_len[i] < 2) return fail(RETINA_EINVAL, "axis_len[%d] = %d < 2", i, axis_len[i]);
        if (!axis_nodes[i]) return fail(RETINA_EINVAL, "axis_nodes[%d] is NULL", i);
        cells *= axis_len[i];
    }
    if (cells > 0x7fffffffLL) return fail(RETINA_EUNSUPPORTED, "more than 2^31-1 cells per event");
    if (n_events == 0 || capacity == 0) return RETINA_OK;
    if (!response || !peak_index || !peak_count || !peak_theta) return fail(RETINA_EINVAL, "NULL device pointer");
    retina::EstimateArgs a{};
    a.R = response;
    a.n0 = axis_len[0];
    a.n1 = axis_len[1];
    a.n2 = (P == 3) ? axis_len[2] : 1;
    a.P = P;
    a.n_events = n_events;
    a.capacity = capacity;
    a.idx = peak_index;
    a.cnt = peak_count;
    a.nodes0 = axis_nodes[0];
    a.nodes1 = axis_nodes[1];
    a.nodes2 = (P == 3) ? axis_nodes[2] : nullptr;
    a.theta = peak_theta;
    const cudaError_t err = retina::launch_estimate(a, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "retina_estimate_peaks");
    return RETINA_OK;
}

int retina_multistart_optimize(const retina_events *ev, int model, float sigma, int32_t n_seeds,
                               const float *seeds, int32_t n_iters, float step, const float *box_lo,
                               const float *box_hi, float *theta_out, float *response_out,
                               float *grad_out, void *stream) {
    return retina_multistart_optimize_ex(ev, model, sigma, n_seeds, seeds, n_iters, step, box_lo, box_hi, theta_out,
                                         response_out, grad_out, RETINA_MS_DENSE, nullptr, 0, nullptr, stream);
}

size_t retina_multistart_workspace_size(int32_t n_events, int32_t n_seeds, int algorithm) {
    if (algorithm != RETINA_MS_CULLED || n_events <= 0 || n_seeds <= 0) return 0;
    // one size for both culled paths: K4c needs the permutation, K6c also the evaluation counts
    return std::max(retina::multistart_culled_workspace_bytes(n_events, n_seeds),
                    retina::newton_culled_workspace_bytes(n_events, n_seeds));
}

// the dense path's pair count: hits x seeds x (n_iters + 1) passes, added on the device
__global__ void add_dense_pairs_kernel(const int32_t *offsets, int n_events, long long seeds_passes,
                                       unsigned long long *pairs) {
    if (blockIdx.x == 0 && threadIdx.x == 0)
        atomicAdd(pairs, (unsigned long long)(offsets[n_events] - offsets[0]) * (unsigned long long)seeds_passes);
}

int retina_multistart_optimize_ex(const retina_events *ev, int model, float sigma, int32_t n_seeds,
                                  const float *seeds, int32_t n_iters, float step, const float *box_lo,
                                  const float *box_hi, float *theta_out, float *response_out, float *grad_out,
                                  int algorithm, void *workspace, size_t workspace_bytes,
                                  unsigned long long *pairs_evaluated, void *stream) {
    g_last_error[0] = 0;
    if (algorithm != RETINA_MS_DENSE && algorithm != RETINA_MS_CULLED)
        return fail(RETINA_EINVAL, "unknown multi-start algorithm %d", algorithm);
    int st = check_events(ev);
    if (st) return st;
    const int P = model_P(model);
    if (P < 0) return fail(RETINA_EINVAL, "unknown model %d", model);
    if (!finite_pos(sigma)) return fail(RETINA_EINVAL, "sigma must be finite and > 0");
    if (n_seeds < 0) return fail(RETINA_EINVAL, "n_seeds < 0");
    if (n_iters < 0) return fail(RETINA_EINVAL, "n_iters < 0");
    if (!std::isfinite(step)) return fail(RETINA_EINVAL, "step is not finite");
    if (!box_lo || !box_hi) return fail(RETINA_EINVAL, "box_lo/box_hi is NULL");
    for (int i = 0; i < P; ++i)
        if (!(box_lo[i] <= box_hi[i])) return fail(RETINA_EINVAL, "box_lo[%d] > box_hi[%d]", i, i);
    if (ev->n_events == 0 || n_seeds == 0) return RETINA_OK;
    if (!seeds || !theta_out || !response_out) return fail(RETINA_EINVAL, "NULL device pointer");
    if ((long long)ev->n_events * n_seeds * P > 0x7fffffffffffLL)
        return fail(RETINA_EUNSUPPORTED, "too many seeds");
    retina::MultistartArgs a{};
    a.offsets = ev->offsets;
    a.hits = reinterpret_cast<const float4 *>(ev->hits);
    a.z_ref = ev->z_ref;
    a.negK = neg_k(sigma);
    a.c2 = c2_of(sigma);
    a.sk = sk_of(sigma);
    a.c2s = c2s_of(sigma);
    a.step = step;
    for (int i = 0; i < 3; ++i) {
        a.lo[i] = (i < P) ? box_lo[i] : 0.f;
        a.hi[i] = (i < P) ? box_hi[i] : 0.f;
    }
    a.n_seeds = n_seeds;
    a.n_iters = n_iters;
    a.seeds = seeds;
    a.theta_out = theta_out;
    a.R_out = response_out;
    a.grad_out = grad_out;
    a.cap = stage_cap(ev->max_event_hits, 4096);
    cudaError_t err;
    if (algorithm == RETINA_MS_CULLED) {
        if (!retina::multistart_culled_ok(model, n_seeds))
            return fail(RETINA_EUNSUPPORTED, "RETINA_MS_CULLED: SLOPE2 / SLOPE3 with n_seeds <= 16384 only");
        const size_t need = retina_multistart_workspace_size(ev->n_events, n_seeds, algorithm);
        if (!workspace || workspace_bytes < need)
            return fail(RETINA_EINVAL, "workspace of %zu bytes needed (got %zu)", need, workspace_bytes);
        err = retina::launch_multistart_culled(model, a, ev->n_events, static_cast<int32_t *>(workspace),
                                               pairs_evaluated, (cudaStream_t)stream);
    } else {
        err = retina::launch_multistart(model, a, ev->n_events, (cudaStream_t)stream);
        if (err == cudaSuccess && pairs_evaluated) {
            add_dense_pairs_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(ev->offsets, ev->n_events,
                                                                      (long long)n_seeds * (n_iters + 1),
                                                                      pairs_evaluated);
            err = cudaGetLastError();
        }
    }
    if (err != cudaSuccess) return cuda_fail(err, "retina_multistart_optimize");
    return RETINA_OK;
}

int retina_multistart_newton(const retina_events *ev, int model, int32_t n_seeds, const float *seeds,
                             int32_t n_steps, const float *sigmas, const float *etas, float final_sigma,
                             int32_t max_halvings, const float *box_lo, const float *box_hi, float *theta_out,
                             float *response_out, float *grad_out, void *stream) {
    return retina_multistart_newton_ex(ev, model, n_seeds, seeds, n_steps, sigmas, etas, final_sigma, max_halvings,
                                       box_lo, box_hi, theta_out, response_out, grad_out, nullptr, stream);
}

int retina_multistart_newton_ex(const retina_events *ev, int model, int32_t n_seeds, const float *seeds,
                                int32_t n_steps, const float *sigmas, const float *etas, float final_sigma,
                                int32_t max_halvings, const float *box_lo, const float *box_hi, float *theta_out,
                                float *response_out, float *grad_out, int32_t *evals_out, void *stream) {
    return retina_multistart_newton_ex2(ev, model, n_seeds, seeds, n_steps, sigmas, etas, final_sigma, max_halvings,
                                        box_lo, box_hi, theta_out, response_out, grad_out, evals_out, RETINA_MS_DENSE,
                                        nullptr, 0, nullptr, stream);
}

int retina_multistart_newton_ex2(const retina_events *ev, int model, int32_t n_seeds, const float *seeds,
                                 int32_t n_steps, const float *sigmas, const float *etas, float final_sigma,
                                 int32_t max_halvings, const float *box_lo, const float *box_hi, float *theta_out,
                                 float *response_out, float *grad_out, int32_t *evals_out, int algorithm,
                                 void *workspace, size_t workspace_bytes, unsigned long long *pairs_evaluated,
                                 void *stream) {
    g_last_error[0] = 0;
    if (algorithm != RETINA_MS_DENSE && algorithm != RETINA_MS_CULLED)
        return fail(RETINA_EINVAL, "unknown multi-start algorithm %d", algorithm);
    int st = check_events(ev);
    if (st) return st;
    const int P = model_P(model);
    if (P < 0) return fail(RETINA_EINVAL, "unknown model %d", model);
    if (model == RETINA_LINE2D) return fail(RETINA_EUNSUPPORTED, "Newton update implemented for SLOPE2/SLOPE3");
    if (n_seeds < 0) return fail(RETINA_EINVAL, "n_seeds < 0");
    if (n_steps < 0) return fail(RETINA_EINVAL, "n_steps < 0");
    if (n_steps > retina::kMaxNewtonSteps) return fail(RETINA_EUNSUPPORTED, "n_steps > %d", retina::kMaxNewtonSteps);
    if (max_halvings < 0) return fail(RETINA_EINVAL, "max_halvings < 0");
    // the queued line search forms 2^-k from the exponent field: exact for k <= 126 (normal floats)
    if (max_halvings > 126) return fail(RETINA_EUNSUPPORTED, "max_halvings %d > 126", max_halvings);
    if (n_steps > 0 && (!sigmas || !etas)) return fail(RETINA_EINVAL, "sigmas/etas is NULL");
    for (int j = 0; j < n_steps; ++j) {
        if (!finite_pos(sigmas[j])) return fail(RETINA_EINVAL, "sigmas[%d] must be finite and > 0", j);
        if (!std::isfinite(etas[j])) return fail(RETINA_EINVAL, "etas[%d] is not finite", j);
    }
    if (!finite_pos(final_sigma)) return fail(RETINA_EINVAL, "final_sigma must be finite and > 0");
    if (!box_lo || !box_hi) return fail(RETINA_EINVAL, "box_lo/box_hi is NULL");
    for (int i = 0; i < P; ++i)
        if (!(box_lo[i] <= box_hi[i])) return fail(RETINA_EINVAL, "box_lo[%d] > box_hi[%d]", i, i);
    if (ev->n_events == 0 || n_seeds == 0) return RETINA_OK;
    if (!seeds || !theta_out || !response_out) return fail(RETINA_EINVAL, "NULL device pointer");
    retina::NewtonArgs a{};
    a.offsets = ev->offsets;
    a.hits = reinterpret_cast<const float4 *>(ev->hits);
    a.z_ref = ev->z_ref;
    a.n_seeds = n_seeds;
    a.seeds = seeds;
    a.n_steps = n_steps;
    for (int j = 0; j < n_steps; ++j) {
        a.negK[j] = neg_k(sigmas[j]);
        a.c2[j] = c2_of(sigmas[j]);
        a.eta[j] = etas[j];
    }
    a.final_negK = neg_k(final_sigma);
    a.final_c2 = c2_of(final_sigma);
    a.max_halvings = max_halvings;
    for (int i = 0; i < 3; ++i) {
        a.lo[i] = (i < P) ? box_lo[i] : 0.f;
        a.hi[i] = (i < P) ? box_hi[i] : 0.f;
    }
    a.theta_out = theta_out;
    a.R_out = response_out;
    a.grad_out = grad_out;
    a.evals_out = evals_out;
    a.reuse_final = (grad_out == nullptr && n_steps > 0 && a.negK[n_steps - 1] == a.final_negK) ? 1 : 0;
    a.cap = stage_cap(ev->max_event_hits, 4096);
    cudaError_t err;
    if (algorithm == RETINA_MS_CULLED) {
        if (!retina::multistart_culled_ok(model, n_seeds))
            return fail(RETINA_EUNSUPPORTED, "RETINA_MS_CULLED: n_seeds <= 16384 only");
        const size_t need = retina_multistart_workspace_size(ev->n_events, n_seeds, algorithm);
        if (!workspace || workspace_bytes < need)
            return fail(RETINA_EINVAL, "workspace of %zu bytes needed (got %zu)", need, workspace_bytes);
        err = retina::launch_newton_culled(model, a, ev->n_events, static_cast<int32_t *>(workspace), pairs_evaluated,
                                           (cudaStream_t)stream);
    } else {
        err = retina::launch_newton(model, a, ev->n_events, pairs_evaluated, (cudaStream_t)stream);
    }
    if (err != cudaSuccess) return cuda_fail(err, "retina_multistart_newton");
    return RETINA_OK;
}

int retina_merge_tracks(int32_t n_events, int32_t n_seeds, int32_t P, const float *theta,
                        const float *response, const float *radius, float threshold, int32_t capacity,
                        float *track_theta, float *track_response, int32_t *track_seed,
                        int32_t *track_size, int32_t *track_count, void *stream) {
    g_last_error[0] = 0;
    if (n_events < 0) return fail(RETINA_EINVAL, "n_events < 0");
    if (n_seeds < 0) return fail(RETINA_EINVAL, "n_seeds < 0");
    if (P != 2 && P != 3) return fail(RETINA_EINVAL, "P must be 2 or 3 (got %d)", P);
    if (capacity < 0) return fail(RETINA_EINVAL, "capacity < 0");
    if (!radius) return fail(RETINA_EINVAL, "radius is NULL");
    for (int i = 0; i < P; ++i)
        if (!(radius[i] >= 0.f) || !std::isfinite(radius[i]))
            return fail(RETINA_EINVAL, "radius[%d] must be finite and >= 0", i);
    if (std::isnan(threshold)) return fail(RETINA_EINVAL, "threshold is NaN");
    if (n_seeds > RETINA_MERGE_MAX_SEEDS)
        return fail(RETINA_EUNSUPPORTED, "n_seeds %d > %d", n_seeds, RETINA_MERGE_MAX_SEEDS);
    if (n_events == 0) return RETINA_OK;
    if (!track_count || (n_seeds > 0 && (!theta || !response)) ||
        (capacity > 0 && (!track_theta || !track_response || !track_seed || !track_size)))
        return fail(RETINA_EINVAL, "NULL device pointer");
    retina::MergeArgs a{};
    a.n_seeds = n_seeds;
    a.P = P;
    a.theta = theta;
    a.R = response;
    for (int i = 0; i < 3; ++i) a.radius[i] = (i < P) ? (double)radius[i] : 0.0;
    a.threshold = threshold;
    a.capacity = capacity;
    a.t_theta = track_theta;
    a.t_R = track_response;
    a.t_seed = track_seed;
    a.t_size = track_size;
    a.t_count = track_count;
    const cudaError_t err = retina::launch_merge(a, n_events, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "retina_merge_tracks");
    return RETINA_OK;
}

int retina_pack_results(int32_t n_events, int32_t P, int32_t keep, const int32_t *peak_index,
                        const float *peak_value, const int32_t *peak_count, int32_t peak_capacity,
                        const float *track_theta, const float *track_response, const int32_t *track_size,
                        const int32_t *track_count, int32_t track_capacity, const uint32_t *header,
                        uint32_t *out, void *stream) {
    g_last_error[0] = 0;
    if (n_events < 0) return fail(RETINA_EINVAL, "n_events < 0");
    if (P != 2 && P != 3) return fail(RETINA_EINVAL, "P must be 2 or 3 (got %d)", P);
    if (keep < 0 || peak_capacity < 0 || track_capacity < 0) return fail(RETINA_EINVAL, "negative keep/capacity");
    if (!header || !out) return fail(RETINA_EINVAL, "header or out is NULL");
    if (n_events > 0 && (!peak_count || !track_count)) return fail(RETINA_EINVAL, "NULL count pointer");
    if (n_events > 0 && keep > 0 &&
        ((peak_capacity > 0 && (!peak_index || !peak_value)) ||
         (track_capacity > 0 && (!track_theta || !track_response || !track_size))))
        return fail(RETINA_EINVAL, "NULL device pointer");
    retina::PackArgs a{};
    a.n_events = n_events;
    a.P = P;
    a.keep = keep;
    a.peak_index = peak_index;
    a.peak_value = peak_value;
    a.peak_count = peak_count;
    a.peak_cap = peak_capacity;
    a.track_theta = track_theta;
    a.track_response = track_response;
    a.track_size = track_size;
    a.track_count = track_count;
    a.track_cap = track_capacity;
    for (int i = 0; i < RETINA_PACK_HEADER; ++i) a.header[i] = header[i];
    a.out = out;
    const cudaError_t err = retina::launch_pack(a, (cudaStream_t)stream);
    if (err != cudaSuccess) return cuda_fail(err, "retina_pack_results");
    return RETINA_OK;
}

}  // extern "C"
