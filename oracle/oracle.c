/* oracle.c -- fp64 CPU oracle for the Artificial Retina hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1709_08610_b200/) never imports, links or calls it,
 * and this file shares no code, header, table or constant with it.
 *
 * What it computes is the plain definition, in double precision, on the same
 * fp32 input arrays the GPU receives (promoted exactly to double):
 *
 *   Eq. (1)  (Sec. 2)   R(theta) = sum_k exp(-s(x_k, theta)^2 / sigma^2)
 *   Eq. (2)              R_ij = R(theta_ij) on a lattice of units
 *   grad R    chain rule through s^2 (derivation below)
 *   step iii             "select clusters of activated units" read as
 *                                       strict local maxima over existing neighbours
 *                                       with R >= R0 (reading Z6)
 *   Alg. 1         multi-start: theta^0 = seeds, q fixed updates
 *                                       theta <- clamp(theta + eta grad R) (reading Z7),
 *                                       cluster, per cluster keep the highest R >= R0
 *                                       (readings Z9, Z10)
 *
 * Distance s ("the distance between hit x and the line defined by
 * parameters theta"; PAPER.md:74 / 195 "euclidean distance in corresponding
 * detector planes"):
 *   model 0  LINE2D  theta = (a, b),        hit (x, y):    s   = y - (a x + b)
 *   model 1  SLOPE2  theta = (tx, ty),      hit (x, y, z): s^2 = (x - tx d)^2 + (y - ty d)^2, d = z - z_ref
 *   model 2  SLOPE3  theta = (tx, ty, z0),  hit (x, y, z): s^2 = (x - tx d)^2 + (y - ty d)^2, d = z - z0
 *
 * Sums run sequentially in hit-array order.  No cutoff on far hits.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ORA_LINE2D = 0, ORA_SLOPE2 = 1, ORA_SLOPE3 = 2 };

static int model_P(int model) { return model == ORA_SLOPE3 ? 3 : 2; }

int ora_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the following parallel loops (bench.py times the oracle on 1 core and on
 * all cores); no effect on any result. */
void ora_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* R, grad R and A_i = sum_k |d_i t_k| at one theta (Eq. 1 and its gradient).
 *
 * With t_k = exp(-s_k^2 / sigma^2):
 *   LINE2D: s = y - a x - b;  dR/da = (2/sigma^2) sum t s x;  dR/db = (2/sigma^2) sum t s
 *   SLOPE2/3: s_x = x - tx d, s_y = y - ty d
 *           dR/dtx = (2/sigma^2) sum t s_x d;  dR/dty = (2/sigma^2) sum t s_y d
 *   SLOPE3:   dR/dz0 = -(2/sigma^2) sum t (s_x tx + s_y ty)      (d = z - z0, dd/dz0 = -1)
 * grad and A may be NULL. */
void ora_point(int model, const float *hits, int n, double z_ref, const double *theta,
               double sigma, double *R_out, double *grad, double *A) {
    const double inv_s2 = 1.0 / (sigma * sigma);
    const int P = model_P(model);
    double R = 0.0, g[3] = {0, 0, 0}, a[3] = {0, 0, 0};
    for (int k = 0; k < n; ++k) {
        const double x = hits[4 * k + 0], y = hits[4 * k + 1], z = hits[4 * k + 2];
        double s2, dg[3] = {0, 0, 0};
        if (model == ORA_LINE2D) {
            const double s = y - (theta[0] * x + theta[1]);
            s2 = s * s;
            dg[0] = s * x;
            dg[1] = s;
        } else {
            const double d = (model == ORA_SLOPE3) ? z - theta[2] : z - z_ref;
            const double sx = x - theta[0] * d, sy = y - theta[1] * d;
            s2 = sx * sx + sy * sy;
            dg[0] = sx * d;
            dg[1] = sy * d;
            if (model == ORA_SLOPE3) dg[2] = -(sx * theta[0] + sy * theta[1]);
        }
        const double t = exp(-s2 * inv_s2);
        R += t;
        for (int i = 0; i < P; ++i) {
            g[i] += t * dg[i];
            a[i] += fabs(t * dg[i]);
        }
    }
    *R_out = R;
    for (int i = 0; i < P; ++i) {
        if (grad) grad[i] = 2.0 * inv_s2 * g[i];
        if (A) A[i] = 2.0 * inv_s2 * a[i];
    }
}

/* Eq. (2): R at every node tuple of every event.  out is [E][n0][n1] (P = 2) or
 * [E][n2][n0][n1] (P = 3: one [n0][n1] plane per z0 node; reading Z37), last axis fastest.
 * nodes_k are fp32 node tables (reading Z4). */
void ora_grid(int model, int n_events, const int32_t *offsets, const float *hits, double z_ref,
              double sigma, const int32_t *axis_len, const float *nodes0, const float *nodes1,
              const float *nodes2, double *out) {
    const int P = model_P(model);
    const int64_t n0 = axis_len[0], n1 = axis_len[1], n2 = (P == 3) ? axis_len[2] : 1;
    const int64_t per_event = n0 * n1 * n2;
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int64_t e = 0; e < n_events; ++e) {
        for (int64_t i = 0; i < n0; ++i) {
            const float *h = hits + 4 * (int64_t)offsets[e];
            const int n = offsets[e + 1] - offsets[e];
            for (int64_t j = 0; j < n1; ++j) {
                for (int64_t l = 0; l < n2; ++l) {
                    double th[3] = {nodes0[i], nodes1[j], P == 3 ? nodes2[l] : 0.0};
                    double R;
                    ora_point(model, h, n, z_ref, th, sigma, &R, NULL, NULL);
                    out[e * per_event + (l * n0 + i) * n1 + j] = R;
                }
            }
        }
    }
}

/* Step (iii), reading Z6: cell c is a peak iff R_c >= R0 and
 * R_c > R_n for every EXISTING neighbour n (3^P - 1 of them in the interior;
 * boundary cells have fewer).  The rule is symmetric in the axes, so it is applied to the
 * grid as a dense row-major array: axis_len is its shape in memory order ((n2, n0, n1) for a
 * P = 3 grid, reading Z37).  Peaks are listed in ascending linear index;
 * count is the true count, entries past `capacity` are dropped. */
void ora_peaks(const double *grid, int n_events, int P, const int32_t *axis_len, double threshold,
               int capacity, int32_t *peak_index, double *peak_value, int32_t *peak_count) {
    const int64_t n0 = axis_len[0], n1 = axis_len[1], n2 = (P == 3) ? axis_len[2] : 1;
    const int64_t per_event = n0 * n1 * n2;
#pragma omp parallel for schedule(dynamic)
    for (int e = 0; e < n_events; ++e) {
        const double *g = grid + e * per_event;
        int32_t cnt = 0;
        for (int64_t i = 0; i < n0; ++i)
            for (int64_t j = 0; j < n1; ++j)
                for (int64_t l = 0; l < n2; ++l) {
                    const int64_t c = (i * n1 + j) * n2 + l;
                    const double v = g[c];
                    int is_peak = v >= threshold;
                    for (int di = -1; di <= 1 && is_peak; ++di)
                        for (int dj = -1; dj <= 1 && is_peak; ++dj)
                            for (int dl = (P == 3 ? -1 : 0); dl <= (P == 3 ? 1 : 0) && is_peak; ++dl) {
                                if (di == 0 && dj == 0 && dl == 0) continue;
                                const int64_t ii = i + di, jj = j + dj, ll = l + dl;
                                if (ii < 0 || ii >= n0 || jj < 0 || jj >= n1 || ll < 0 || ll >= n2) continue;
                                if (!(v > g[(ii * n1 + jj) * n2 + ll])) is_peak = 0;
                            }
                    if (is_peak) {
                        if (cnt < capacity) {
                            peak_index[(int64_t)e * capacity + cnt] = (int32_t)c;
                            peak_value[(int64_t)e * capacity + cnt] = v;
                        }
                        ++cnt;
                    }
                }
        peak_count[e] = cnt;
    }
}

/* Algorithm 1, lines "for j = 1..q: compute R, grad R; theta^j := update[...]"
 * with update = fixed-step ascent clamped to the prior box
 * (reading Z7): theta^{j+1} = clamp(theta^j + eta grad R(theta^j)).  Returns
 * theta^n, R(theta^n) and grad R(theta^n) (grad_out may be NULL). */
void ora_multistart(int model, int n_events, const int32_t *offsets, const float *hits,
                    double z_ref, double sigma, int n_seeds, const float *seeds, int n_iters,
                    double step, const double *box_lo, const double *box_hi, double *theta_out,
                    double *R_out, double *grad_out) {
    const int P = model_P(model);
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
    for (int64_t e = 0; e < n_events; ++e) {
        for (int64_t s = 0; s < n_seeds; ++s) {
            const float *h = hits + 4 * (int64_t)offsets[e];
            const int n = offsets[e + 1] - offsets[e];
            const int64_t id = (int64_t)e * n_seeds + s;
            double th[3] = {0, 0, 0}, g[3], R;
            for (int i = 0; i < P; ++i) th[i] = seeds[id * P + i];
            for (int j = 0; j < n_iters; ++j) {
                ora_point(model, h, n, z_ref, th, sigma, &R, g, NULL);
                for (int i = 0; i < P; ++i) {
                    double v = th[i] + step * g[i];
                    if (v < box_lo[i]) v = box_lo[i];
                    if (v > box_hi[i]) v = box_hi[i];
                    th[i] = v;
                }
            }
            ora_point(model, h, n, z_ref, th, sigma, &R, g, NULL);
            for (int i = 0; i < P; ++i) theta_out[id * P + i] = th[i];
            R_out[id] = R;
            if (grad_out)
                for (int i = 0; i < P; ++i) grad_out[id * P + i] = g[i];
        }
    }
}

/* Algorithm 1, "cluster solutions; for each cluster select solution with
 * highest response and above threshold R0", readings Z9/Z10:
 *   keep items with R >= R0; order them by (R desc, theta lexicographic asc,
 *   seed index asc); scan that order: an item joins the EARLIEST-created leader
 *   L with max_i |theta_i - L_i| <= r_i, else it founds a new leader.  Leaders
 *   are emitted in creation order with their cluster sizes. */
typedef struct { const double *theta; const double *R; int P; } merge_ctx;

static int merge_cmp(const void *pa, const void *pb, void *vctx) {
    const merge_ctx *c = (const merge_ctx *)vctx;
    const int32_t a = *(const int32_t *)pa, b = *(const int32_t *)pb;
    if (c->R[a] > c->R[b]) return -1;
    if (c->R[a] < c->R[b]) return 1;
    for (int i = 0; i < c->P; ++i) {
        if (c->theta[(int64_t)a * c->P + i] < c->theta[(int64_t)b * c->P + i]) return -1;
        if (c->theta[(int64_t)a * c->P + i] > c->theta[(int64_t)b * c->P + i]) return 1;
    }
    return (a < b) ? -1 : (a > b);
}

void ora_merge(int n_events, int n_seeds, int P, const double *theta, const double *R,
               const double *radius, double threshold, int capacity, double *track_theta,
               double *track_R, int32_t *track_seed, int32_t *track_size, int32_t *track_count,
               int32_t *member) {
    /* member (may be NULL): [n_events][n_seeds], the creation ordinal of the leader each seed
     * joined, -1 below the threshold (bookkeeping for the T6 comparator; no arithmetic). */
#pragma omp parallel for schedule(dynamic)
    for (int e = 0; e < n_events; ++e) {
        const double *th = theta + (int64_t)e * n_seeds * P;
        const double *r = R + (int64_t)e * n_seeds;
        int32_t *items = (int32_t *)malloc(sizeof(int32_t) * (n_seeds > 0 ? n_seeds : 1));
        int32_t *leader = (int32_t *)malloc(sizeof(int32_t) * (n_seeds > 0 ? n_seeds : 1));
        int32_t *size = (int32_t *)malloc(sizeof(int32_t) * (n_seeds > 0 ? n_seeds : 1));
        int m = 0;
        int32_t *mem = member ? member + (int64_t)e * n_seeds : NULL;
        for (int s = 0; s < n_seeds; ++s) {
            if (mem) mem[s] = -1;
            if (r[s] >= threshold) items[m++] = s;
        }
        merge_ctx ctx = {th, r, P};
        qsort_r(items, m, sizeof(int32_t), merge_cmp, &ctx);
        int L = 0;
        for (int q = 0; q < m; ++q) {
            const int s = items[q];
            int found = -1;
            for (int l = 0; l < L && found < 0; ++l) {
                int inside = 1;
                for (int i = 0; i < P; ++i)
                    if (!(fabs(th[(int64_t)s * P + i] - th[(int64_t)leader[l] * P + i]) <= radius[i])) inside = 0;
                if (inside) found = l;
            }
            if (found >= 0) {
                size[found] += 1;
            } else {
                leader[L] = s;
                size[L] = 1;
                found = L++;
            }
            if (mem) mem[s] = found;
        }
        for (int l = 0; l < L && l < capacity; ++l) {
            const int64_t o = (int64_t)e * capacity + l;
            for (int i = 0; i < P; ++i) track_theta[o * P + i] = th[(int64_t)leader[l] * P + i];
            track_R[o] = r[leader[l]];
            track_seed[o] = leader[l];
            track_size[o] = size[l];
        }
        track_count[e] = L;
        free(items);
        free(leader);
        free(size);
    }
}

/* Step (iv) ("for each cluster estimate track parameters"), reading Z21
 * (SPEC.md:292-300): per peak and per axis, the vertex of the parabola through the values at
 * the peak cell and its two neighbours along that axis, in units of the local half-spacing
 * (node[c+1] - node[c-1]) / 2; the cell centre when a neighbour is missing (lattice
 * boundary) or the three points are not strictly concave.  The vertex of a parabola through
 * (-1, a), (0, b), (1, c) is at (a - c) / (2 (a - 2 b + c)). */
void ora_estimate(const double *grid, int n_events, int P, const int32_t *axis_len, const float *nodes0,
                  const float *nodes1, const float *nodes2, const int32_t *peak_index,
                  const int32_t *peak_count, int capacity, double *theta) {
    /* axis_len in parameter order (tx, ty[, z0]); cell (i, j[, l]) sits at (l n0 + i) n1 + j (Z37) */
    const int64_t n[3] = {axis_len[0], axis_len[1], P == 3 ? axis_len[2] : 1};
    const int64_t per_event = n[0] * n[1] * n[2];
    const int64_t stride[3] = {n[1], 1, n[0] * n[1]};
    const float *nodes[3] = {nodes0, nodes1, nodes2};
    for (int e = 0; e < n_events; ++e) {
        const int cnt = peak_count[e] < capacity ? peak_count[e] : capacity;
        for (int p = 0; p < cnt; ++p) {
            const int64_t c = peak_index[(int64_t)e * capacity + p];
            const int64_t ci[3] = {(c / n[1]) % n[0], c % n[1], c / (n[0] * n[1])};
            const double *g = grid + e * per_event;
            for (int i = 0; i < P; ++i) {
                double t = nodes[i][ci[i]];
                if (ci[i] > 0 && ci[i] < n[i] - 1) {
                    const double a = g[c - stride[i]], b = g[c], cc = g[c + stride[i]];
                    const double den = 2.0 * (a - 2.0 * b + cc);
                    if (den < 0.0) {
                        double delta = (a - cc) / den;
                        if (delta > 0.5) delta = 0.5;
                        if (delta < -0.5) delta = -0.5;
                        t += delta * 0.5 * ((double)nodes[i][ci[i] + 1] - (double)nodes[i][ci[i] - 1]);
                    }
                }
                theta[((int64_t)e * capacity + p) * P + i] = t;
            }
        }
    }
}

/* ------------------------------------------------------------------------------------------
 * NEXT #1: the paper's own update: Truncated Newton steps on R with the
 * Hessian (Algorithm 1 line "compute response R, gradient grad R and Hessian H R",
 * PAPER.md:150) and a per-step bandwidth schedule sigma_1..sigma_q.
 *
 * R, gradient and Hessian at one theta, by the chain rule through f = s^2 / sigma^2 with the
 * residual vector r(theta) = (s) (LINE2D) or (s_x, s_y) (SLOPE2/3):
 *     t_k = exp(-f_k),  d_a f = (2/sigma^2) sum_c r_c d_a r_c,
 *     d_ab f = (2/sigma^2) sum_c (d_a r_c d_b r_c + r_c d_ab r_c),
 *     dR/d_a = -sum_k t_k d_a f_k,   H_ab = sum_k t_k (d_a f_k d_b f_k - d_ab f_k).
 * Residual derivatives: LINE2D r = y - a x - b: dr = (-x, -1).  SLOPE2 r = (x - tx d, y - ty d),
 * d = z - z_ref: d r_x/d tx = -d, d r_y/d ty = -d.  SLOPE3 d = z - z0: additionally
 * d r_x/d z0 = tx, d r_y/d z0 = ty, d2 r_x/(d tx d z0) = 1, d2 r_y/(d ty d z0) = 1.
 * H is row-major P x P; grad, H may be NULL. */
void ora_point_hess(int model, const float *hits, int n, double z_ref, const double *theta, double sigma,
                    double *R_out, double *grad, double *H) {
    const int P = model_P(model);
    const double c = 2.0 / (sigma * sigma);
    double R = 0.0, g[3] = {0, 0, 0}, h[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (int k = 0; k < n; ++k) {
        const double x = hits[4 * k + 0], y = hits[4 * k + 1], z = hits[4 * k + 2];
        double r[2] = {0, 0}, J[2][3] = {{0, 0, 0}, {0, 0, 0}}, K2[2][3][3];
        memset(K2, 0, sizeof(K2));
        int nr;
        if (model == ORA_LINE2D) {
            nr = 1;
            r[0] = y - (theta[0] * x + theta[1]);
            J[0][0] = -x;
            J[0][1] = -1.0;
        } else {
            nr = 2;
            const double d = (model == ORA_SLOPE3) ? z - theta[2] : z - z_ref;
            r[0] = x - theta[0] * d;
            r[1] = y - theta[1] * d;
            J[0][0] = -d;
            J[1][1] = -d;
            if (model == ORA_SLOPE3) {
                J[0][2] = theta[0];
                J[1][2] = theta[1];
                K2[0][0][2] = K2[0][2][0] = 1.0;
                K2[1][1][2] = K2[1][2][1] = 1.0;
            }
        }
        double f = 0.0;
        for (int q = 0; q < nr; ++q) f += r[q] * r[q];
        f /= sigma * sigma;
        const double t = exp(-f);
        double df[3] = {0, 0, 0};
        for (int a = 0; a < P; ++a)
            for (int q = 0; q < nr; ++q) df[a] += c * r[q] * J[q][a];
        R += t;
        for (int a = 0; a < P; ++a) {
            g[a] -= t * df[a];
            for (int b = 0; b < P; ++b) {
                double d2f = 0.0;
                for (int q = 0; q < nr; ++q) d2f += c * (J[q][a] * J[q][b] + r[q] * K2[q][a][b]);
                h[a * 3 + b] += t * (df[a] * df[b] - d2f);
            }
        }
    }
    *R_out = R;
    for (int a = 0; a < P; ++a) {
        if (grad) grad[a] = g[a];
        if (H)
            for (int b = 0; b < P; ++b) H[a * P + b] = h[a * 3 + b];
    }
}

/* Truncated-Newton direction for MAXIMISING R (reading Z23): conjugate gradients on
 * (-H) p = g, at most P iterations (exact for a positive-definite -H), stopped at a direction
 * of non-positive curvature d^T (-H) d <= 0: the iterate built so far is kept, or, at the first
 * iteration, the fixed-step gradient direction p = eta g (reading Z24). */
/* splitmix64 of (key, seed, counter) mapped to a uniform double in [-1, 1] (test perturbations) */
static double unit_hash(uint64_t key, int64_t id, uint64_t c) {
    uint64_t z = key * 0x9E3779B97F4A7C15ull ^ ((uint64_t)id * 0xBF58476D1CE4E5B9ull) ^ (c * 0x94D049BB133111EBull);
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

typedef struct {        /* per-seed decision bookkeeping (T5n attribution; no effect by default) */
    double *margin;     /* smallest relative margin of any decision taken                       */
    double *log;        /* nullable: margin of decision k at log[k], k < log_len                 */
    int log_len;
    int count;          /* decisions taken so far                                               */
    const uint8_t *flip; /* nullable: decision k's outcome is inverted when flip[k] != 0, k < log_len */
} decisions;

/* Records one discrete decision's relative margin m and returns its outcome, inverted when it
 * is the decision the caller asked to flip (test attribution of fp32/fp64 near-ties). */
static int decide(decisions *dc, int outcome, double m) {
    if (m < *dc->margin) *dc->margin = m;
    if (dc->log && dc->count < dc->log_len) dc->log[dc->count] = m;
    const int flip = dc->flip && dc->count < dc->log_len && dc->flip[dc->count];
    dc->count++;
    return flip ? !outcome : outcome;
}

static void tn_direction(int P, const double *g, const double *H, double eta, double *p, decisions *dc) {
    double x[3] = {0, 0, 0}, r[3], d[3], Ad[3];
    double hs = 0.0;  /* scale of H for the curvature-decision margin (diagnostic only) */
    for (int a = 0; a < P * P; ++a) hs = fabs(H[a]) > hs ? fabs(H[a]) : hs;
    double rr = 0.0;
    for (int a = 0; a < P; ++a) {
        r[a] = g[a];
        d[a] = g[a];
        rr += g[a] * g[a];
    }
    const double rr0 = rr;
    int it;
    for (it = 0; it < P && rr > 0.0; ++it) {
        double curv = 0.0;
        for (int a = 0; a < P; ++a) {
            Ad[a] = 0.0;
            for (int b = 0; b < P; ++b) Ad[a] -= H[a * P + b] * d[b];
            curv += d[a] * Ad[a];
        }
        double dd = 0.0;
        for (int a = 0; a < P; ++a) dd += d[a] * d[a];
        const double m = (dd > 0.0 && hs > 0.0) ? fabs(curv) / (dd * hs) : 1.0;
        /* a flipped decision never divides by a zero curvature */
        if (!decide(dc, curv > 0.0, m) || curv == 0.0) {
            if (it == 0)
                for (int a = 0; a < P; ++a) x[a] = eta * g[a];
            break;
        }
        const double alpha = rr / curv;
        double rr_new = 0.0;
        for (int a = 0; a < P; ++a) {
            x[a] += alpha * d[a];
            r[a] -= alpha * Ad[a];
            rr_new += r[a] * r[a];
        }
        if (rr_new <= 1e-24 * rr0) break;
        const double beta = rr_new / rr;
        for (int a = 0; a < P; ++a) d[a] = r[a] + beta * d[a];
        rr = rr_new;
    }
    for (int a = 0; a < P; ++a) p[a] = x[a];
}

/* Algorithm 1 with update[.] = one Truncated-Newton step per
 * optimisation step j = 1..q at bandwidth sigma_j, with Armijo
 * backtracking on R (reading Z25: c1 = 1e-4, alpha = 1, 1/2, ..., at most max_halvings
 * halvings; theta is clamped to the prior box at every trial; no accepted trial leaves theta
 * unchanged).  Returns theta^q, R(theta^q) and grad R(theta^q) at final_sigma.
 * perturb_eps > 0 (test attribution only): every evaluated R, grad R and H entry is multiplied by
 * 1 + perturb_eps u, u uniform in [-1, 1] from a counter hash of (perturb_key, seed, evaluation),
 * i.e. the oracle runs with arithmetic errors of the GPU's size (T5n "arithmetic sensitivity").
 * flip (nullable; test attribution only): [seed][log_len] flags; decision k of a seed (CG curvature
 * tests and Armijo tests, numbered in the order taken) has its outcome inverted when flag k is set;
 * decision_log (nullable) receives each decision's relative margin ([seed][log_len], -1 = unused).
 * margin_out (nullable; diagnostic for the T5 near-tie rule, no effect on the result): per seed,
 * the smallest relative margin of any discrete decision taken -- |R_t - (R_0 + c1 alpha g.p)| /
 * R_0 for the Armijo tests and |d^T H d| / (|d|^2 max|H|) for the CG curvature tests.
 * evals_out (nullable): per seed, the response evaluations Algorithm 1 spent on it, in the
 * paper's cost unit: q evaluations with gradient and Hessian, every line-search
 * trial, and the final evaluation, i.e. q + sum_j (trials of step j) + 1 -- without the final one
 * when it would repeat an evaluation already made (no gradient wanted, grad_out == NULL, and
 * final_sigma == sigmas[q-1]: R(theta^q) at that sigma is the last accepted trial's value, or the
 * last Hessian-mode evaluation's if no trial was accepted; Z36). */
void ora_newton(int model, int n_events, const int32_t *offsets, const float *hits, double z_ref, int n_seeds,
                const float *seeds, int n_steps, const double *sigmas, const double *etas, double final_sigma,
                int max_halvings, const double *box_lo, const double *box_hi, double *theta_out,
                double *R_out, double *grad_out, double *margin_out, int32_t *evals_out, const uint8_t *flip,
                double *decision_log, int log_len, double perturb_eps, uint64_t perturb_key) {
    const int P = model_P(model);
#pragma omp parallel for collapse(2) schedule(dynamic, 16)
    for (int64_t e = 0; e < n_events; ++e) {
        for (int64_t s = 0; s < n_seeds; ++s) {
            const float *h = hits + 4 * (int64_t)offsets[e];
            const int n = offsets[e + 1] - offsets[e];
            const int64_t id = e * n_seeds + s;
            double th[3] = {0, 0, 0}, g[3], H[9], p[3], R0, Rt, tt[3], margin = 1.0;
            int32_t evals = 0;
            decisions dc = {&margin, decision_log ? decision_log + id * log_len : NULL, log_len, 0,
                            flip ? flip + id * log_len : NULL};
            if (dc.log)
                for (int k = 0; k < log_len; ++k) dc.log[k] = -1.0;
            for (int a = 0; a < P; ++a) th[a] = seeds[id * P + a];
            uint64_t pc = 0; /* perturbation counter of this seed */
            for (int j = 0; j < n_steps; ++j) {
                ora_point_hess(model, h, n, z_ref, th, sigmas[j], &R0, g, H);
                ++evals;
                if (perturb_eps > 0.0) {
                    R0 *= 1.0 + perturb_eps * unit_hash(perturb_key, id, pc++);
                    for (int a = 0; a < P; ++a) g[a] *= 1.0 + perturb_eps * unit_hash(perturb_key, id, pc++);
                    for (int a = 0; a < P; ++a)
                        for (int b = a; b < P; ++b) {
                            H[a * P + b] *= 1.0 + perturb_eps * unit_hash(perturb_key, id, pc++);
                            H[b * P + a] = H[a * P + b];
                        }
                }
                tn_direction(P, g, H, etas[j], p, &dc);
                double slope = 0.0;
                for (int a = 0; a < P; ++a) slope += g[a] * p[a];
                double alpha = 1.0;
                for (int k = 0; k <= max_halvings; ++k, alpha *= 0.5) {
                    for (int a = 0; a < P; ++a) {
                        double v = th[a] + alpha * p[a];
                        if (v < box_lo[a]) v = box_lo[a];
                        if (v > box_hi[a]) v = box_hi[a];
                        tt[a] = v;
                    }
                    ora_point_hess(model, h, n, z_ref, tt, sigmas[j], &Rt, NULL, NULL);
                    ++evals;
                    if (perturb_eps > 0.0) Rt *= 1.0 + perturb_eps * unit_hash(perturb_key, id, pc++);
                    const double m = fabs(Rt - (R0 + 1e-4 * alpha * slope)) / (R0 > 1e-6 ? R0 : 1e-6);
                    if (decide(&dc, Rt >= R0 + 1e-4 * alpha * slope, m)) {
                        for (int a = 0; a < P; ++a) th[a] = tt[a];
                        break;
                    }
                }
            }
            ora_point_hess(model, h, n, z_ref, th, final_sigma, &R0, g, NULL);
            for (int a = 0; a < P; ++a) theta_out[id * P + a] = th[a];
            R_out[id] = R0;
            if (grad_out)
                for (int a = 0; a < P; ++a) grad_out[id * P + a] = g[a];
            if (margin_out) margin_out[id] = margin;
            if (evals_out) {
                const int reuse = !grad_out && n_steps > 0 && (float)sigmas[n_steps - 1] == (float)final_sigma;
                evals_out[id] = evals + (reuse ? 0 : 1);
            }
        }
    }
}
