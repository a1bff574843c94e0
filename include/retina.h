/* retina.h -- C ABI of the B200 (sm_100a) Artificial Retina hot path.
 *
 * arXiv 1709.08610, "Numerical optimization for Artificial Retina Algorithm".
 * The four entry points of the hot path, one per step of the method:
 *
 *   retina_grid_response        Eq. (1)-(2), PAPER.md:36-39 (Sec. 2) and step (ii),
 *                               R_ij = sum_k exp(-s(x_k, theta_ij)^2 / sigma^2)
 *                               for every unit of a lattice, for every event of a batch.
 *   retina_find_peaks           step (iii), "select clusters of activated
 *                               units", read as strict local maxima (Z6).
 *   retina_multistart_optimize  Algorithm 1: seeds theta^0 (drawn by the
 *                               caller from the prior), a FIXED number
 *                               of updates theta <- clamp(theta + step grad R) (PAPER.md:136,
 *                               151; Z7); returns theta^n, R(theta^n), grad R(theta^n).
 *   retina_merge_tracks         Algorithm 1: "cluster solutions; for each
 *                               cluster select solution with highest response and above
 *                               threshold R0" (Z9, Z10).
 * and the "next" rows built on them:
 *   retina_grid_response_ex     the same grid with an explicit kernel choice (_ex2: + pairs contracted);
 *   retina_find_peaks_ws        step (iii) by many CTAs per event (caller workspace);
 *   retina_estimate_peaks       step (iv): sub-cell parameter estimate per peak;
 *   retina_multistart_optimize_ex  the same update loop, optionally evaluating only the pairs that
 *                               can contribute (bit-identical results; RETINA_MS_CULLED);
 *   retina_multistart_newton    Algorithm 1 with the paper's Truncated-Newton update and sigma
 *   (_ex, _ex2)                 schedule, PAPER.md:213-216 (+ per-seed evaluation counts; _ex2:
 *                               optionally culled like the update loop, bit-identical results);
 *   retina_pack_results         the per-rank record of the one multi-GPU result gather.
 *
 * Track models and the distance s:
 *   RETINA_LINE2D  P=2, theta=(a, b),       hit (x, y, -, -):  s   = y - (a x + b)
 *   RETINA_SLOPE2  P=2, theta=(tx, ty),     hit (x, y, z, -):  s^2 = (x - tx d)^2 + (y - ty d)^2, d = z - z_ref
 *   RETINA_SLOPE3  P=3, theta=(tx, ty, z0), hit (x, y, z, -):  s^2 = (x - tx d)^2 + (y - ty d)^2, d = z - z0
 *
 * Conventions (all entry points):
 *  - Bulk data are DEVICE pointers (CUDA global memory of the current device); small
 *    descriptors (axis lengths, node-table pointer arrays, box, radius) are HOST pointers.
 *  - Ownership: every buffer is caller-owned.  The library never allocates device
 *    memory, never frees, and keeps no pointer after the call returns.
 *  - Asynchrony: every call only enqueues kernels on `stream` (a cudaStream_t passed as
 *    void*; NULL = legacy default stream) and never synchronizes.  Safe to call from
 *    several host threads on different streams.
 *  - Errors: host-checkable problems return RETINA_EINVAL synchronously and launch
 *    nothing (NULL pointers, n_events < 0, sigma <= 0 or non-finite, unknown model or
 *    model/P mismatch, axis_len < 2, capacity < 0, n_iters < 0, n_seeds < 0, box_lo >
 *    box_hi, radius < 0).  Sizes the kernels do not support return RETINA_EUNSUPPORTED
 *    (e.g. n_seeds > RETINA_MERGE_MAX_SEEDS in merge, or > 2^31 cells per event).  A
 *    failed launch returns RETINA_ECUDA.  retina_last_error() gives a thread-local
 *    message for the last non-OK return.
 *  - Capacity overflow is NOT an error: *_count holds the TRUE count, and entries past
 *    `capacity` are dropped; the caller sees it after synchronizing.
 *  - Determinism: outputs are bit-identical for identical inputs (no float atomics, fixed
 *    per-thread accumulation order, deterministic compaction and sort).
 *  - Precision: fp32 storage and arithmetic, exp lowered to ex2.approx with the
 *    log2(e)/sigma^2 scale applied after squaring; residuals formed with exact
 *    products (FMA) and, where a difference of coordinates is inexact (z - z_ref,
 *    z - z0, y - a x), as double-float pairs.  The tensor-core grid kernels
 *    split every fp32 factor exactly into tf32 or scaled fp16 parts and accumulate the
 *    products in fp32, for fp32-level accuracy.
 *  - There is no CPU fallback: without a CUDA device every call returns RETINA_ECUDA.
 */
#ifndef RETINA_H
#define RETINA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { RETINA_OK = 0, RETINA_EINVAL = 1, RETINA_EUNSUPPORTED = 2, RETINA_ECUDA = 3 };
enum { RETINA_LINE2D = 0, RETINA_SLOPE2 = 1, RETINA_SLOPE3 = 2 };

#define RETINA_MERGE_MAX_SEEDS 16384

/* A batch of events in CSR form ("a set of hits"; "An event
 * consists of N_e coordinates (x, y, z) of triggered pixels").
 *   offsets:  device int32 [n_events + 1], offsets[0] = 0, non-decreasing; event e owns
 *             hits offsets[e] .. offsets[e+1]-1.
 *   hits:     device float [4 * offsets[n_events]], (x, y, z, 0) per hit, 16-byte aligned
 *             (may be NULL only when the batch holds no hit).
 *             Hits sorted by z within an event make SLOPE3 multi-start faster (it
 *             re-forms z - z0 only when z changes); any order gives the same results
 *             up to fp32 summation order being the array order.
 *   z_ref:    SLOPE2 only: z of the pattern origin (0 in every BASELINE config).
 *   max_event_hits: optional HOST-side upper bound on hits per event (0 = unknown).  It
 *             only sizes the shared-memory hit buffer (events that fit stay resident
 *             across multi-start iterations); results never depend on it. */
typedef struct {
    int32_t        n_events;
    const int32_t *offsets;
    const float   *hits;
    float          z_ref;
    int32_t        max_event_hits;
} retina_events;

/* Eq. (2): response of every unit of the lattice axis_nodes[0] x ... x axis_nodes[P-1].
 *   model:      RETINA_LINE2D / SLOPE2 (P = 2) or RETINA_SLOPE3 (P = 3).
 *   sigma:      bandwidth of Eq. (1), > 0, in the units of s.
 *   axis_len:   host int32 [P], each >= 2.
 *   axis_nodes: host array [P] of device fp32 [axis_len[i]] node tables (the caller owns
 *               the node values; they are not recomputed, Z4).
 *   response:   device fp32, last axis fastest: [n_events][axis_len[0]][axis_len[1]] for P = 2;
 *               [n_events][axis_len[2]][axis_len[0]][axis_len[1]] for P = 3, i.e. one
 *               (tx, ty) plane per z0 node (Z37; the paper fixes no layout).
 * Returns RETINA_OK, RETINA_EINVAL, RETINA_EUNSUPPORTED or RETINA_ECUDA. */
int retina_grid_response(const retina_events *ev, int model, float sigma,
                         const int32_t *axis_len, const float *const *axis_nodes,
                         float *response, void *stream);

/* Same as retina_grid_response with an explicit kernel choice:
 *   RETINA_GRID_AUTO       tensor (fp16 split) for SLOPE2 and SLOPE3, direct for LINE2D
 *                          (what retina_grid_response uses);
 *   RETINA_GRID_DIRECT     one MUFU.EX2 per (unit, hit) pair (all models);
 *   RETINA_GRID_SEPARABLE  SLOPE2/SLOPE3 only: exp(-s^2/sigma^2) = e_x(tx, hit) e_y(ty, hit)
 *                          exactly, so the grid is a dense contraction over hits, done with
 *                          FFMA2 on the CUDA cores (RETINA_EUNSUPPORTED for LINE2D, whose
 *                          residual does not split);
 *   RETINA_GRID_TENSOR     SLOPE2 / SLOPE3 (one GEMM per z0): the same contraction on the tcgen05 tensor cores with a
 *                          3xTF32 split (fp32-level accuracy), accumulators in TMEM;
 *   RETINA_GRID_TENSOR_F16 SLOPE2 / SLOPE3: the same contraction on kind::f16 with an exact scaled fp16 hi/lo
 *                          split of every factor (fp32-level accuracy, half the MMA work of 3xTF32), by
 *                          persistent CTA pairs (cta_group::2, M = 256) with double-buffered TMEM
 *                          accumulators (a three-part split gives one accumulator per tile);
 *   RETINA_GRID_TENSOR_F16_PAIR    the same split by one CTA pair per 256 x 256 tile (two accumulators:
 *                          hi.hi and hi.lo + lo.hi), non-persistent;
 *   RETINA_GRID_TENSOR_F16_SINGLE  the same by one CTA per 128 x 256 tile (no cluster);
 *   RETINA_GRID_TENSOR_F16_CULLED  RETINA_GRID_TENSOR_F16 where every 256 x 256 tile contracts only the hits
 *                          that can reach it: a conservative bound keeps a hit unless K s^2 > 128 for every
 *                          (tx, ty) of the tile, i.e. unless each of its products e_x e_y is below 2^-128 --
 *                          below fp32's normal range -- for every cell; the grid stays within the T1
 *                          tolerance of the dense one, not bit-identical (the tensor-core sums group the
 *                          remaining hits differently).  Row pitches that are not a multiple of 16 bytes run
 *                          the dense kernel. */
enum { RETINA_GRID_AUTO = 0, RETINA_GRID_DIRECT = 1, RETINA_GRID_SEPARABLE = 2, RETINA_GRID_TENSOR = 3,
       RETINA_GRID_TENSOR_F16 = 4, RETINA_GRID_TENSOR_F16_PAIR = 5, RETINA_GRID_TENSOR_F16_SINGLE = 6,
       RETINA_GRID_TENSOR_F16_CULLED = 7 };
int retina_grid_response_ex(const retina_events *ev, int model, float sigma,
                            const int32_t *axis_len, const float *const *axis_nodes,
                            float *response, int algorithm, void *stream);
/* retina_grid_response_ex that also ADDS to *pairs_evaluated (device uint64, may be NULL) the
 * (unit, hit) pairs the kernel contracted: hits x cells for every algorithm but
 * RETINA_GRID_TENSOR_F16_CULLED, which counts, per tile, its cells x the hits it kept. */

int retina_grid_response_ex2(const retina_events *ev, int model, float sigma,
                             const int32_t *axis_len, const float *const *axis_nodes,
                             float *response, int algorithm, unsigned long long *pairs_evaluated,
                             void *stream);

/* Step (iii) on a response grid (any fp32 grid of that shape):
 * cell c is reported iff response[c] >= threshold and response[c] > response[n] for every
 * EXISTING neighbour n of its 3^P - 1 neighbourhood (cells on the lattice boundary have
 * fewer neighbours; equal neighbours -- plateaus -- give no peak).
 *   response:    device fp32 [n_events][cells] in the layout retina_grid_response writes; P in
 *                {2, 3}; axis_len host int32 [P] in parameter order, as there.  The rule is
 *                symmetric in the axes and is applied in memory order.
 *   capacity:    entries per event of the output lists, >= 0.
 *   peak_index:  device int32 [n_events][capacity], flat offset of the cell within its event's
 *                grid ((l n0 + i) n1 + j for P = 3), ascending.
 *   peak_value:  device fp32  [n_events][capacity], response at that cell.
 *   peak_count:  device int32 [n_events], TRUE number of peaks (may exceed capacity). */
int retina_find_peaks(const float *response, int32_t n_events, int32_t P,
                      const int32_t *axis_len, float threshold, int32_t capacity,
                      int32_t *peak_index, float *peak_value, int32_t *peak_count,
                      void *stream);

/* Same result as retina_find_peaks, computed by many CTAs per event (slabs of cells: a scan
 * pass that counts each slab's peaks and keeps the first 1,024 of them, then a write pass that
 * copies them to the deterministic prefix of the slab counts -- a slab with more peaks is
 * scanned again) using a caller-owned DEVICE workspace of at least
 * retina_find_peaks_workspace_size() bytes (its contents on entry do not matter).  Faster than
 * one CTA per event whenever the events do not fill whole waves of CTAs (cfg3: 2.20 vs 2.50 ms per
 * 2,048 events; 256^3 grids: much faster).  workspace_bytes too small -> RETINA_EINVAL. */
size_t retina_find_peaks_workspace_size(int32_t n_events, int32_t P, const int32_t *axis_len);
int retina_find_peaks_ws(const float *response, int32_t n_events, int32_t P, const int32_t *axis_len,
                         float threshold, int32_t capacity, int32_t *peak_index, float *peak_value,
                         int32_t *peak_count, void *workspace, size_t workspace_bytes, void *stream);

/* Step (iv), "for each cluster estimate track parameters" (Z21):
 * for every listed peak, per axis i, the vertex of the parabola through the peak cell and its
 * two neighbours along i,
 *     delta = (R- - R+) / (2 (R- - 2 R0 + R+)),  theta_i = node_i[c_i] + delta (node_i[c_i+1] - node_i[c_i-1]) / 2,
 * falling back to the cell centre on the lattice boundary (a neighbour missing) or when the
 * curvature is not negative; |delta| <= 1/2 (a strict maximum keeps the vertex in its cell).
 *   response:    device fp32 grid, as given to retina_find_peaks.
 *   axis_len, axis_nodes: as in retina_grid_response (host arrays; device node tables).
 *   peak_index, peak_count, capacity: the outputs of retina_find_peaks.
 *   peak_theta:  device fp32 [n_events][capacity][P]; entries >= min(count, capacity) untouched. */
int retina_estimate_peaks(const float *response, int32_t n_events, int32_t P,
                          const int32_t *axis_len, const float *const *axis_nodes,
                          const int32_t *peak_index, const int32_t *peak_count, int32_t capacity,
                          float *peak_theta, void *stream);

/* Algorithm 1 update loop with update = fixed-step gradient ascent clamped to the prior
 * box (Z7).  For every (event e, seed i):
 *     theta^0 = seeds[e][i];  theta^{j+1} = clamp(theta^j + step * grad R(theta^j)),
 *     j = 0 .. n_iters-1, clamp per axis to [box_lo, box_hi];
 *   then theta_out = theta^n, response_out = R(theta^n), grad_out = grad R(theta^n).
 * n_iters = 0 evaluates R and grad R at the seeds (BASELINE configs[0] "grad R at 256
 * random theta").
 *   seeds:        device fp32 [n_events][n_seeds][P].
 *   box_lo/hi:    host fp32 [P].
 *   theta_out:    device fp32 [n_events][n_seeds][P]; may alias seeds.
 *   response_out: device fp32 [n_events][n_seeds].
 *   grad_out:     device fp32 [n_events][n_seeds][P], or NULL (then the last pass
 *                 evaluates R only). */
int retina_multistart_optimize(const retina_events *ev, int model, float sigma,
                               int32_t n_seeds, const float *seeds, int32_t n_iters,
                               float step, const float *box_lo, const float *box_hi,
                               float *theta_out, float *response_out, float *grad_out,
                               void *stream);

/* retina_multistart_optimize with an explicit algorithm:
 *   RETINA_MS_DENSE   evaluates every (seed, hit) pair of every pass (what retina_multistart_optimize
 *                     does; workspace unused);
 *   RETINA_MS_CULLED  SLOPE2 / SLOPE3 (RETINA_EUNSUPPORTED for LINE2D): the SAME results bit for bit,
 *                     evaluating only the pairs that can contribute.  With ex2.approx.ftz a pair
 *                     whose exponent -K s^2 is below -126 adds exactly +0 to R and to the gradient
 *                     sums; the seeds of each event are ordered along a Morton curve of theta so
 *                     that every warp's 256 seeds cover a small box, and per pass each warp skips the
 *                     hits that a conservative bound puts beyond K s^2 > 128 for all of them, visiting
 *                     the others in hit order with K4's arithmetic.  Needs a DEVICE workspace of at
 *                     least retina_multistart_workspace_size() bytes (8 per seed and event: the
 *                     per-event permutation, and for retina_multistart_newton_ex2 the evaluation
 *                     counts between its step launches; contents on entry do not matter);
 *                     n_seeds <= 16,384 (the per-event sort runs in shared memory).  Events larger
 *                     than the hit stage run the dense passes.
 *   pairs_evaluated:  device uint64 or NULL: the (seed, hit) pairs actually evaluated are ADDED to
 *                     it (all pairs for RETINA_MS_DENSE).
 * Other arguments as retina_multistart_optimize. */
enum { RETINA_MS_DENSE = 0, RETINA_MS_CULLED = 1 };
size_t retina_multistart_workspace_size(int32_t n_events, int32_t n_seeds, int algorithm);
int retina_multistart_optimize_ex(const retina_events *ev, int model, float sigma,
                                  int32_t n_seeds, const float *seeds, int32_t n_iters,
                                  float step, const float *box_lo, const float *box_hi,
                                  float *theta_out, float *response_out, float *grad_out,
                                  int algorithm, void *workspace, size_t workspace_bytes,
                                  unsigned long long *pairs_evaluated, void *stream);

/* Algorithm 1 with the paper's own update (Z22-Z25): q = n_steps
 * Truncated-Newton steps, step j at bandwidth sigmas[j] with R, grad R and the Hessian H R from
 * one pass over the hits, direction by conjugate gradients on (-H) p = grad R
 * (<= P iterations; stopped at non-positive curvature, or p = etas[j] grad R at the first
 * iteration), then backtracking alpha = 1, 1/2, ... (<= max_halvings halvings) accepting the
 * first clamp(theta + alpha p) with R >= R(theta) + 1e-4 alpha grad R . p (else theta stays).
 * Returns theta^q, R(theta^q) and grad R(theta^q) at final_sigma.  The direction is solved in
 * fp64 from the fp32-accumulated grad R and H (SLOPE3's Hessian mixes slope and mm scales).
 * SLOPE2 / SLOPE3 only (RETINA_EUNSUPPORTED for LINE2D); n_steps <= 16; max_halvings <= 126
 * (RETINA_EUNSUPPORTED above: 2^-k is formed exactly only for normal floats).
 *   sigmas, etas: host fp32 [n_steps]; other arguments as retina_multistart_optimize. */
int retina_multistart_newton(const retina_events *ev, int model, int32_t n_seeds, const float *seeds,
                             int32_t n_steps, const float *sigmas, const float *etas, float final_sigma,
                             int32_t max_halvings, const float *box_lo, const float *box_hi,
                             float *theta_out, float *response_out, float *grad_out, void *stream);

/* retina_multistart_newton plus the paper's cost accounting (cost in
 * units of one response evaluation): evals_out, device int32 [n_events][n_seeds] or NULL,
 * receives per seed the response evaluations Algorithm 1 spent on it -- n_steps evaluations
 * with gradient and Hessian, every line-search trial, and the final evaluation
 * (= n_steps + sum_j trials_j + 1).  When grad_out is NULL and final_sigma equals
 * sigmas[n_steps-1], R(theta^q) is the value the last step already computed at that point (its
 * accepted trial, or its Hessian-mode evaluation when no trial was accepted): no final pass runs
 * and the count has no final term.  Identical results otherwise. */
int retina_multistart_newton_ex(const retina_events *ev, int model, int32_t n_seeds, const float *seeds,
                                int32_t n_steps, const float *sigmas, const float *etas, float final_sigma,
                                int32_t max_halvings, const float *box_lo, const float *box_hi,
                                float *theta_out, float *response_out, float *grad_out, int32_t *evals_out,
                                void *stream);

/* retina_multistart_newton_ex with an explicit algorithm (as retina_multistart_optimize_ex):
 *   RETINA_MS_DENSE   every pass visits every hit (what retina_multistart_newton_ex does);
 *   RETINA_MS_CULLED  the SAME results bit for bit (theta, R, grad R and evals_out), each warp
 *                     visiting only the hits that can contribute: one launch per Newton step, before
 *                     which the seeds of each event are re-ordered along a Morton curve of their
 *                     current theta; in every pass (Hessian mode, each line-search trial pass, the
 *                     final pass) a warp lists, in hit order, the hits a conservative bound keeps
 *                     within K_j s^2 <= 128 of the box of the points it evaluates (K_j = 1/sigma_j^2
 *                     of that pass); the others would add exactly +0 under ex2.approx.ftz.
 *                     Needs a DEVICE workspace of at least retina_multistart_workspace_size(n_events,
 *                     n_seeds, RETINA_MS_CULLED) bytes; n_seeds <= 16,384.  Events larger than the
 *                     hit stage run the dense passes, and so does RETINA_SLOPE3 (its wide early
 *                     sigma_j keep nearly every hit in reach); the results are the same either way.
 *   pairs_evaluated:  device uint64 or NULL: RETINA_MS_DENSE ADDS evaluations x hits (every
 *                     evaluation visits every hit); RETINA_MS_CULLED adds the (seed, hit) pairs its
 *                     passes visited for real seeds (including the line search's speculative
 *                     halvings, which evals_out does not count). */
int retina_multistart_newton_ex2(const retina_events *ev, int model, int32_t n_seeds, const float *seeds,
                                 int32_t n_steps, const float *sigmas, const float *etas, float final_sigma,
                                 int32_t max_halvings, const float *box_lo, const float *box_hi,
                                 float *theta_out, float *response_out, float *grad_out, int32_t *evals_out,
                                 int algorithm, void *workspace, size_t workspace_bytes,
                                 unsigned long long *pairs_evaluated, void *stream);

/* Algorithm 1 "cluster solutions ... select highest response above R0" per event:
 *   keep seeds with response >= threshold; order them by (response descending, theta
 *   lexicographic ascending, seed index ascending); scan that order: a seed joins the
 *   EARLIEST-created leader L with |theta_i - L_i| <= radius[i] for every axis i
 *   (differences formed exactly, in fp64), otherwise it founds a new leader.
 *   theta, response: device fp32 [n_events][n_seeds][P] and [n_events][n_seeds].
 *   radius:          host fp32 [P], >= 0.  n_seeds <= RETINA_MERGE_MAX_SEEDS.
 *   track_theta:     device fp32 [n_events][capacity][P], leaders in creation order
 *                    (= response descending).
 *   track_response:  device fp32 [n_events][capacity].
 *   track_seed:      device int32 [n_events][capacity], leader's seed index.
 *   track_size:      device int32 [n_events][capacity], number of above-threshold members.
 *   track_count:     device int32 [n_events], TRUE number of clusters. */
int retina_merge_tracks(int32_t n_events, int32_t n_seeds, int32_t P, const float *theta,
                        const float *response, const float *radius, float threshold,
                        int32_t capacity, float *track_theta, float *track_response,
                        int32_t *track_seed, int32_t *track_size, int32_t *track_count,
                        void *stream);

/* The per-rank result record of the one multi-GPU gather (north
 * star: "one NCCL gather over NVLink for found tracks and timings only"): packs the first
 * `keep` peaks and tracks of every event and the rank's header into a fixed-size buffer of
 * 32-bit words that the caller all-gathers (fp32 fields as bit patterns, so the record is exact):
 *   out[0 .. RETINA_PACK_HEADER): header[] as given, except out[3] = sum of peak_count and
 *       out[4] = sum of track_count (computed on the device; saturate at 2^32 - 1);
 *   then per event e, RETINA_PACK_WORDS(P, keep) words: peak_count[e], track_count[e],
 *       keep peak indices (-1 past min(count, capacity)), keep peak values (fp32 bits, 0 past),
 *       keep x (track_theta[P], track_response (fp32 bits), track_size) (0 past).
 *   n_events >= 0, P in {2, 3}, keep >= 0, capacities >= 0; peak_* / track_* are the device
 *   outputs of retina_find_peaks and retina_merge_tracks (layouts as there); header: host
 *   [RETINA_PACK_HEADER] (rank, event base, n_events, -, -, pairs_grid/1e9 and
 *   pairs_multistart/1e9 as fp32 bits, 0); out: device, RETINA_PACK_HEADER +
 *   n_events * RETINA_PACK_WORDS(P, keep) words, caller-owned.  NULL pointers or negative sizes
 *   -> RETINA_EINVAL.  Deterministic. */
#define RETINA_PACK_HEADER 8
#define RETINA_PACK_WORDS(P, keep) (2 + 2 * (keep) + (keep) * ((P) + 2))
int retina_pack_results(int32_t n_events, int32_t P, int32_t keep, const int32_t *peak_index,
                        const float *peak_value, const int32_t *peak_count, int32_t peak_capacity,
                        const float *track_theta, const float *track_response, const int32_t *track_size,
                        const int32_t *track_count, int32_t track_capacity, const uint32_t *header,
                        uint32_t *out, void *stream);

/* Static description of a status code. */
const char *retina_status_string(int status);
/* Thread-local detail for the last non-OK return of the calling thread ("" if none). */
const char *retina_last_error(void);
/* Library version string, e.g. "retina-b200 0.1 sm_100a". */
const char *retina_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RETINA_H */
