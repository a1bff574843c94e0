// kernels.cuh -- argument blocks and host launchers of the retina kernels (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace retina {

enum { kLine2D = 0, kSlope2 = 1, kSlope3 = 2 };

struct GridArgs {
    const int32_t *offsets;
    const float4 *hits;
    float z_ref;
    float negK;  // -log2(e) / sigma^2, rounded once from fp64 on the host
    int n0, n1, n2;
    const float *nodes0, *nodes1, *nodes2;
    float *R;
    int cap;     // float4 slots of the shared-memory hit stage
    int e_base;
    unsigned long long *pairs;  // culled tensor grid: (unit, hit) pairs contracted are added here (or NULL)
};

struct MultistartArgs {
    const int32_t *offsets;
    const float4 *hits;
    float z_ref;
    float negK;   // -log2(e) / sigma^2
    float c2;     // 2 / sigma^2 (gradient prefactor)
    float sk;     // sqrt(log2(e)) / sigma (SLOPE3: residuals are formed already scaled by it)
    float c2s;    // c2 / sk (SLOPE3 gradient prefactor for the scaled residual sums)
    float step;
    float lo[3], hi[3];
    int n_seeds;
    int n_iters;
    const float *seeds;
    float *theta_out, *R_out, *grad_out;
    int cap;
    int compact;  // SLOPE3: hits staged as (x, y) pairs + a per-plane z table (cap float2 slots)
    int e_base;
};

constexpr int kMaxNewtonSteps = 16;

struct NewtonArgs {
    const int32_t *offsets;
    const float4 *hits;
    float z_ref;
    int n_seeds;
    const float *seeds;
    int n_steps;
    float negK[kMaxNewtonSteps];  // -log2(e)/sigma_j^2
    float c2[kMaxNewtonSteps];    // 2/sigma_j^2
    float eta[kMaxNewtonSteps];   // gradient fallback step per optimisation step
    float final_negK, final_c2;
    int max_halvings;
    float lo[3], hi[3];
    float *theta_out, *R_out, *grad_out;
    int32_t *evals_out;  // nullable: response evaluations per seed (q + line-search trials [+ 1 final])
    int reuse_final;     // no final pass: final sigma == last sigma and no gradient output
    int cap;
    int e_base;
    // steps [j_begin, j_end) in this launch; first: theta from seeds (else theta_out) and fresh counts
    // (else nev_ws); last: the final pass and every output (else theta_out and nev_ws only)
    int j_begin, j_end, first, last;
    int32_t *nev_ws;  // K6c: [n_events][n_seeds] evaluation counts between step launches
};

struct PeakArgs {
    const float *R;
    int n0, n1, n2;  // grid dims in MEMORY order, n2 fastest (P = 3: z0, tx, ty -- DESIGN.md Z37); n2 = 1 for P = 2
    int P;
    float threshold;
    int capacity;
    int32_t *idx;
    float *val;
    int32_t *cnt;
    int e_base;
};

struct MergeArgs {
    int n_seeds;
    int P;
    const float *theta;
    const float *R;
    double radius[3];
    float threshold;
    int capacity;
    float *t_theta;
    float *t_R;
    int32_t *t_seed;
    int32_t *t_size;
    int32_t *t_count;
    int e_base;
};

struct EstimateArgs {
    const float *R;
    int n0, n1, n2;  // node counts in parameter order (tx, ty, z0); n2 = 1 for P = 2
    int P;
    int n_events;
    int capacity;
    const int32_t *idx;
    const int32_t *cnt;
    const float *nodes0, *nodes1, *nodes2;
    float *theta;
};

struct PackArgs {
    int n_events, P, keep;
    const int32_t *peak_index;
    const float *peak_value;
    const int32_t *peak_count;
    int peak_cap;
    const float *track_theta;
    const float *track_response;
    const int32_t *track_size;
    const int32_t *track_count;
    int track_cap;
    uint32_t header[8];  // RETINA_PACK_HEADER words from the caller; [3], [4] are filled on the device
    uint32_t *out;
};

cudaError_t launch_pack(const PackArgs &a, cudaStream_t stream);
cudaError_t launch_estimate(const EstimateArgs &a, cudaStream_t stream);
cudaError_t launch_grid_response(int model, const GridArgs &a, int n_events, cudaStream_t stream);
cudaError_t launch_grid_separable(int model, const GridArgs &a, int n_events, cudaStream_t stream);
cudaError_t launch_grid_tensor(int model, const GridArgs &a, int n_events, cudaStream_t stream);
cudaError_t launch_grid_tensor16(int model, const GridArgs &a, int n_events, cudaStream_t stream);
cudaError_t launch_grid_tensor16p(int model, const GridArgs &a, int n_events, cudaStream_t stream, bool cull = false);
cudaError_t launch_grid_tensor16x2(int model, const GridArgs &a, int n_events, cudaStream_t stream);
cudaError_t launch_newton(int model, const NewtonArgs &a, int n_events, unsigned long long *pairs_evaluated,
                          cudaStream_t stream);
// K6c (newton.cu): the same results as K6, evaluating only the pairs that can contribute; ws holds
// the per-event Morton permutation and the evaluation counts (newton_culled_workspace_bytes)
size_t newton_culled_workspace_bytes(long long n_events, int n_seeds);
cudaError_t launch_newton_culled(int model, const NewtonArgs &a, int n_events, int32_t *ws,
                                 unsigned long long *pairs_evaluated, cudaStream_t stream);
// K4c-sort: perm[e][q] = caller index of event e's q-th seed along a Morton curve over the box
cudaError_t launch_seed_morton_sort(const float *seeds, int n_seeds, int P, const float (&lo)[3], const float (&hi)[3],
                                    int32_t *perm, int n_events, cudaStream_t stream);
cudaError_t launch_multistart(int model, const MultistartArgs &a, int n_events, cudaStream_t stream);
// K4c (multistart.cu): the same results as K4 for SLOPE2, evaluating only the pairs that can contribute
bool multistart_culled_ok(int model, int n_seeds);
size_t multistart_culled_workspace_bytes(long long n_events, int n_seeds);
cudaError_t launch_multistart_culled(int model, const MultistartArgs &a, int n_events, int32_t *perm,
                                     unsigned long long *pairs_evaluated, cudaStream_t stream);
cudaError_t launch_find_peaks(const PeakArgs &a, int n_events, cudaStream_t stream);
cudaError_t launch_find_peaks_ws(const PeakArgs &a, int n_events, int32_t *ws, cudaStream_t stream);
int peaks_slabs(int cells);
size_t peaks_workspace_bytes(long long n_events, int P, int n0, int n1, int n2);
bool peaks3_brick_ok(int n0, int n1, int n2);
size_t peaks3_workspace_bytes(long long n_events, int n0, int n1, int n2);
cudaError_t launch_find_peaks3_brick(const PeakArgs &a, int n_events, int32_t *ws, cudaStream_t stream);
cudaError_t launch_merge(const MergeArgs &a, int n_events, cudaStream_t stream);

}  // namespace retina
