/*
 * mtsph_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links or loads
 * this file; it is the checker used by tests/, __graft_entry__.smoke() and
 * the cpu_baseline / --impl reference leg of bench.py.  It restates, in
 * plain C (OpenMP on the data-parallel loops, fixed per-particle summation
 * order so results are thread-count independent), the algorithms of the
 * upstream package (paths relative to /root/reference/pkg/src/mtsph):
 *
 *   kernels.py:110      Wendland C2 kernel gradient (anisotropic map)
 *   _accel.py:16        velocity_gradient_gather
 *   _accel.py:34        pair_tensor_divergence
 *   _accel.py:52        pair_tensor_divergence_mapped
 *   _accel.py:76        scalar_difference_flux
 *   _accel.py:171       damping_sweep (+ _damp_single :97, _damp_group :107)
 *   _accel.py:210       conservative_mass_rate
 *   _accel.py:240       porous_stress_rhs
 *   plasticity.py:118   return_map (+ _solve_consistency :89)
 *   solids.py:148/164   kirchhoff_stress / first_pk
 *   scenarios.py:113    NeckingProblem.relax_step (fused here as one call)
 *   solids.py:187       solid_time_step
 *
 * Arrays follow the reference (numpy, C order): vectors (n,d), tensors
 * (n,d,d) row-major, CSR indptr/idx as int64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SQ23 0.81649658092772603273 /* sqrt(2/3) */

/* ---------------------------------------------------------------- tensors */

static double det_n(int d, const double *t) {
    if (d == 1) return t[0];
    if (d == 2) return t[0] * t[3] - t[1] * t[2];
    return t[0] * (t[4] * t[8] - t[5] * t[7])
         - t[1] * (t[3] * t[8] - t[5] * t[6])
         + t[2] * (t[3] * t[7] - t[4] * t[6]);
}

/* adjugate / determinant (reference tensors.py:170 layout) */
static void inv_n(int d, const double *t, double j, double *o) {
    if (d == 1) { o[0] = 1.0 / j; return; }
    if (d == 2) {
        o[0] = t[3] / j; o[1] = -t[1] / j; o[2] = -t[2] / j; o[3] = t[0] / j;
        return;
    }
    o[0] = (t[4] * t[8] - t[5] * t[7]) / j;
    o[1] = (t[2] * t[7] - t[1] * t[8]) / j;
    o[2] = (t[1] * t[5] - t[2] * t[4]) / j;
    o[3] = (t[5] * t[6] - t[3] * t[8]) / j;
    o[4] = (t[0] * t[8] - t[2] * t[6]) / j;
    o[5] = (t[2] * t[3] - t[0] * t[5]) / j;
    o[6] = (t[3] * t[7] - t[4] * t[6]) / j;
    o[7] = (t[1] * t[6] - t[0] * t[7]) / j;
    o[8] = (t[0] * t[4] - t[1] * t[3]) / j;
}

static void matmul_n(int d, const double *a, const double *b, double *o) {
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            double s = 0.0;
            for (int k = 0; k < d; ++k) s += a[r * d + k] * b[k * d + c];
            o[r * d + c] = s;
        }
}

/* a @ b^T */
static void matmul_nt(int d, const double *a, const double *b, double *o) {
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            double s = 0.0;
            for (int k = 0; k < d; ++k) s += a[r * d + k] * b[c * d + k];
            o[r * d + c] = s;
        }
}

/* ----------------------------------------------------------------- kernel */

/* dW/dr_vec of the anisotropic Wendland C2 kernel (kernels.py:110).
 * prefactor = sigma_d / prod(h_axes). */
void or_kernel_grad(int d, const double *rel, const double *h_axes,
                    double prefactor, double *out) {
    double u[3], q2 = 0.0;
    for (int k = 0; k < d; ++k) { u[k] = rel[k] / h_axes[k]; q2 += u[k] * u[k]; }
    double q = sqrt(q2);
    if (!(q > 0.0) || q >= 2.0) { for (int k = 0; k < d; ++k) out[k] = 0.0; return; }
    double t = 1.0 - 0.5 * q;
    double mag = prefactor * (-5.0 * q * t * t * t) / q;
    for (int k = 0; k < d; ++k) out[k] = mag * (u[k] / h_axes[k]);
}

/* --------------------------------------------------------- neighbour build */

/* All pairs i<j with scaled distance |(x_j - x_i)/h| < 2, by a uniform
 * cell grid of edge 2 in the scaled space (reference neighbors.py:77 uses a
 * k-d tree; the set is what matters).  Pairs are emitted sorted by (i, j).
 * Returns the number of pairs, -1 if cap too small, -2 - k on a duplicate
 * position (k = first particle of the coincident pair).
 */
static int cmp_i64pair(const void *a, const void *b) {
    const int64_t *x = (const int64_t *)a, *y = (const int64_t *)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

int64_t or_build_pairs(int64_t n, int d, const double *x, const double *h_axes,
                       int64_t cap, int64_t *pairs /* (cap, 2) */) {
    if (n <= 0) return 0;
    double *u = (double *)malloc(sizeof(double) * n * d);
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < d; ++k) {
            double v = x[i * d + k] / h_axes[k];
            u[i * d + k] = v;
            if (i == 0 || v < lo[k]) lo[k] = v;
            if (i == 0 || v > hi[k]) hi[k] = v;
        }
    int64_t dims[3] = {1, 1, 1};
    for (int k = 0; k < d; ++k) dims[k] = (int64_t)floor((hi[k] - lo[k]) / 2.0) + 1;
    int64_t ncell = dims[0] * dims[1] * dims[2];
    int64_t *cell = (int64_t *)malloc(sizeof(int64_t) * n);
    int64_t *start = (int64_t *)calloc(ncell + 1, sizeof(int64_t));
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * n);
    for (int64_t i = 0; i < n; ++i) {
        int64_t c = 0;
        for (int k = d - 1; k >= 0; --k) {
            int64_t ck = (int64_t)floor((u[i * d + k] - lo[k]) / 2.0);
            if (ck >= dims[k]) ck = dims[k] - 1;
            c = c * dims[k] + ck;
        }
        cell[i] = c;
        start[c + 1]++;
    }
    for (int64_t c = 0; c < ncell; ++c) start[c + 1] += start[c];
    int64_t *fill = (int64_t *)malloc(sizeof(int64_t) * (ncell + 1));
    memcpy(fill, start, sizeof(int64_t) * (ncell + 1));
    for (int64_t i = 0; i < n; ++i) order[fill[cell[i]]++] = i;
    free(fill);

    int64_t np = 0;
    int64_t dup = -1;
    for (int64_t i = 0; i < n && dup < 0; ++i) {
        int64_t ci[3] = {0, 0, 0}, rem = cell[i];
        for (int k = 0; k < d; ++k) { ci[k] = rem % dims[k]; rem /= dims[k]; }
        int64_t span[3] = {0, 0, 0};
        for (int k = 0; k < d; ++k) span[k] = 1;
        for (int64_t o2 = -span[2]; o2 <= span[2]; ++o2)
        for (int64_t o1 = -span[1]; o1 <= span[1]; ++o1)
        for (int64_t o0 = -span[0]; o0 <= span[0]; ++o0) {
            int64_t nc[3] = {ci[0] + o0, ci[1] + o1, ci[2] + o2};
            int ok = 1;
            for (int k = 0; k < 3; ++k) if (nc[k] < 0 || nc[k] >= dims[k]) ok = 0;
            if (!ok) continue;
            int64_t c = (nc[2] * dims[1] + nc[1]) * dims[0] + nc[0];
            for (int64_t s = start[c]; s < start[c + 1]; ++s) {
                int64_t j = order[s];
                if (j <= i) continue;
                double q2 = 0.0;
                for (int k = 0; k < d; ++k) {
                    double du = u[j * d + k] - u[i * d + k];
                    q2 += du * du;
                }
                double q = sqrt(q2);
                if (q == 0.0) { dup = i; break; }
                if (q < 2.0) {
                    if (np >= cap) { np = -1; goto done; }
                    pairs[2 * np] = i; pairs[2 * np + 1] = j; ++np;
                }
            }
        }
    }
done:
    free(u); free(cell); free(start); free(order);
    if (dup >= 0) return -2 - dup;
    if (np > 0) qsort(pairs, (size_t)np, 2 * sizeof(int64_t), cmp_i64pair);
    return np;
}

/* Split runs of equal-key pairs into particle-sharing components, in order
 * of first appearance (neighbors.py:165).  starts has nruns+1 entries.
 * Writes the permutation `order` (npairs) and group starts (<= npairs+1);
 * returns the number of groups, -1 for a run longer than 64 pairs. */
int64_t or_split_runs(int64_t nruns, const int64_t *starts, const int64_t *pi,
                      const int64_t *pj, int64_t *order, int64_t *gstart) {
    int64_t ng = 0;
    int64_t node[128];
    int par[128], ea[64], comp[64], roots[64];
    for (int64_t r = 0; r < nruns; ++r) {
        int64_t lo = starts[r], hi = starts[r + 1];
        int m = (int)(hi - lo);
        if (m == 1) { order[lo] = lo; gstart[ng++] = lo; continue; }
        if (m > 64) return -1;
        int nn = 0;
        for (int k = 0; k < m; ++k) {
            int64_t e[2] = {pi[lo + k], pj[lo + k]};
            int idx[2];
            for (int s = 0; s < 2; ++s) {
                int f = -1;
                for (int t = 0; t < nn; ++t) if (node[t] == e[s]) { f = t; break; }
                if (f < 0) { node[nn] = e[s]; par[nn] = nn; f = nn++; }
                idx[s] = f;
            }
            ea[k] = idx[0];
            int ra = idx[0], rb = idx[1];
            while (par[ra] != ra) ra = par[ra];
            while (par[rb] != rb) rb = par[rb];
            if (ra != rb) { if (ra < rb) par[rb] = ra; else par[ra] = rb; }
        }
        int nc = 0;
        for (int k = 0; k < m; ++k) {
            int x = ea[k];
            while (par[x] != x) x = par[x];
            int f = -1;
            for (int t = 0; t < nc; ++t) if (roots[t] == x) { f = t; break; }
            if (f < 0) { roots[nc] = x; f = nc++; }
            comp[k] = f;
        }
        int64_t w = lo;
        for (int c = 0; c < nc; ++c) {
            gstart[ng++] = w;
            for (int k = 0; k < m; ++k) if (comp[k] == c) order[w++] = lo + k;
        }
    }
    gstart[ng] = starts[nruns];
    return ng;
}

/* --------------------------------------------------------- CSR operators */

void or_velocity_gradient_gather(int64_t n, int d, const double *src,
                                 const int64_t *indptr, const int64_t *idx,
                                 const double *grad, const double *vol,
                                 double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < n; ++a) {
        double acc[9] = {0};
        for (int64_t k = indptr[a]; k < indptr[a + 1]; ++k) {
            int64_t b = idx[k];
            for (int r = 0; r < d; ++r) {
                double dv = vol[b] * (src[b * d + r] - src[a * d + r]);
                for (int c = 0; c < d; ++c) acc[r * d + c] += dv * grad[k * d + c];
            }
        }
        memcpy(out + a * d * d, acc, sizeof(double) * d * d);
    }
}

void or_pair_tensor_divergence(int64_t n, int d, const double *tens,
                               const int64_t *indptr, const int64_t *idx,
                               const double *grad, const double *vol,
                               double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < n; ++a) {
        double acc[3] = {0, 0, 0};
        const double *ta = tens + a * d * d;
        for (int64_t k = indptr[a]; k < indptr[a + 1]; ++k) {
            int64_t b = idx[k];
            const double *tb = tens + b * d * d;
            for (int r = 0; r < d; ++r) {
                double s = 0.0;
                for (int c = 0; c < d; ++c) s += (ta[r * d + c] + tb[r * d + c]) * grad[k * d + c];
                acc[r] += vol[b] * s;
            }
        }
        for (int r = 0; r < d; ++r) out[a * d + r] = acc[r];
    }
}

/* out[a] += sum_b vol_b (tens_a + tens_b) . (amap_a grad_ab) */
void or_pair_tensor_divergence_mapped(int64_t n, int d, const double *tens,
                                      const double *amap, const int64_t *indptr,
                                      const int64_t *idx, const double *grad,
                                      const double *vol, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < n; ++a) {
        const double *ma = amap + a * d * d, *ta = tens + a * d * d;
        for (int64_t k = indptr[a]; k < indptr[a + 1]; ++k) {
            int64_t b = idx[k];
            const double *tb = tens + b * d * d;
            double g[3];
            for (int r = 0; r < d; ++r) {
                double s = 0.0;
                for (int c = 0; c < d; ++c) s += ma[r * d + c] * grad[k * d + c];
                g[r] = s;
            }
            for (int r = 0; r < d; ++r) {
                double s = 0.0;
                for (int c = 0; c < d; ++c) s += (ta[r * d + c] + tb[r * d + c]) * g[c];
                out[a * d + r] += vol[b] * s;
            }
        }
    }
}

/* out[a] = coeff_a sum_b vol_b (sat_a - sat_b) (amap_a grad_ab) */
void or_scalar_difference_flux(int64_t n, int d, const double *sat,
                               const double *coeff, const double *amap,
                               const int64_t *indptr, const int64_t *idx,
                               const double *vol, const double *grad,
                               double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < n; ++a) {
        double acc[3] = {0, 0, 0};
        const double *ma = amap + a * d * d;
        for (int64_t k = indptr[a]; k < indptr[a + 1]; ++k) {
            int64_t b = idx[k];
            double w = vol[b] * (sat[a] - sat[b]);
            for (int r = 0; r < d; ++r) {
                double s = 0.0;
                for (int c = 0; c < d; ++c) s += ma[r * d + c] * grad[k * d + c];
                acc[r] += w * s;
            }
        }
        for (int r = 0; r < d; ++r) out[a * d + r] = acc[r] * coeff[a];
    }
}

/* pair-antisymmetric mass rate (serial: both sides accumulated per pair) */
void or_conservative_mass_rate(int64_t n, int d, const double *flux,
                               const double *amap, int64_t npairs,
                               const int64_t *pi, const int64_t *pj,
                               const double *pgrad, const double *vol,
                               double *out) {
    for (int64_t a = 0; a < n; ++a) out[a] = 0.0;
    for (int64_t k = 0; k < npairs; ++k) {
        int64_t i = pi[k], j = pj[k];
        double acc = 0.0;
        for (int r = 0; r < d; ++r) {
            double s = 0.0;
            for (int c = 0; c < d; ++c)
                s += 0.5 * (amap[i * d * d + r * d + c] + amap[j * d * d + r * d + c]) * pgrad[k * d + c];
            acc += (flux[i * d + r] + flux[j * d + r]) * s;
        }
        double w = vol[i] * vol[j] * acc;
        out[i] -= w;
        out[j] += w;
    }
}

/* mixture stress -> corrected nominal stress tbuf, then pair divergence.
 * Returns the number of particles with J <= 0 (their rows are zeroed). */
int64_t or_porous_stress_rhs(int64_t n, int d, const double *F,
                             const double *pressure, const double *corr,
                             const int64_t *indptr, const int64_t *idx,
                             const double *grad0, const double *vol0,
                             double mu, double lam, double *tbuf,
                             double *jout, double *rate) {
    int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad)
    for (int64_t a = 0; a < n; ++a) {
        const double *f = F + a * d * d;
        double j = det_n(d, f);
        jout[a] = j;
        double *t = tbuf + a * d * d;
        if (j <= 0.0) { for (int k = 0; k < d * d; ++k) t[k] = 0.0; ++bad; continue; }
        double fi[9], e[9], sg[9], pm[9];
        inv_n(d, f, j, fi);
        double tre = 0.0;
        for (int r = 0; r < d; ++r) {
            for (int c = 0; c < d; ++c) {
                double s = 0.0;
                for (int k = 0; k < d; ++k) s += fi[k * d + r] * fi[k * d + c];
                e[r * d + c] = -0.5 * s;
            }
            e[r * d + r] += 0.5;
            tre += e[r * d + r];
        }
        double dia = lam * tre - pressure[a];
        for (int k = 0; k < d * d; ++k) sg[k] = 2.0 * mu * e[k];
        for (int r = 0; r < d; ++r) sg[r * d + r] += dia;
        for (int r = 0; r < d; ++r)
            for (int c = 0; c < d; ++c) {
                double s = 0.0;
                for (int k = 0; k < d; ++k) s += sg[r * d + k] * fi[c * d + k];
                pm[r * d + c] = j * s;
            }
        matmul_n(d, pm, corr + a * d * d, t);
    }
    or_pair_tensor_divergence(n, d, tbuf, indptr, idx, grad0, vol0, rate);
    return bad;
}

/* ------------------------------------------------------------- damping */

static void damp_pair(int d, double *vel, int64_t a, int64_t b, double ca, double cb) {
    double den = 1.0 + ca + cb;
    for (int m = 0; m < d; ++m) {
        double u = (vel[a * d + m] - vel[b * d + m]) / den;
        vel[a * d + m] -= ca * u;
        vel[b * d + m] += cb * u;
    }
}

/* simultaneous backward-Euler solve of one group (nb <= 128 particles) */
static void damp_group(int d, double *vel, const int64_t *pi, const int64_t *pj,
                       const double *pd, const double *imi, const double *imj,
                       double half, int64_t lo, int64_t hi, int64_t *loc,
                       double *A, double *rhs) {
    int nb = 0;
    for (int64_t k = lo; k < hi; ++k) {
        int64_t ends[2] = {pi[k], pj[k]};
        for (int e = 0; e < 2; ++e) {
            int found = 0;
            for (int t = 0; t < nb; ++t) if (loc[t] == ends[e]) { found = 1; break; }
            if (!found) loc[nb++] = ends[e];
        }
    }
    for (int r = 0; r < nb; ++r) {
        for (int c = 0; c < nb; ++c) A[r * 128 + c] = (r == c) ? 1.0 : 0.0;
        for (int m = 0; m < d; ++m) rhs[r * 3 + m] = vel[loc[r] * d + m];
    }
    for (int64_t k = lo; k < hi; ++k) {
        double c = half * pd[k];
        int ia = 0, ib = 0;
        for (int t = 0; t < nb; ++t) {
            if (loc[t] == pi[k]) ia = t;
            if (loc[t] == pj[k]) ib = t;
        }
        double ca = c * imi[k], cb = c * imj[k];
        A[ia * 128 + ia] += ca; A[ia * 128 + ib] -= ca;
        A[ib * 128 + ib] += cb; A[ib * 128 + ia] -= cb;
    }
    for (int col = 0; col < nb - 1; ++col) {
        double piv = A[col * 128 + col];
        for (int r = col + 1; r < nb; ++r) {
            double f = A[r * 128 + col] / piv;
            if (f != 0.0) {
                for (int c = col; c < nb; ++c) A[r * 128 + c] -= f * A[col * 128 + c];
                for (int m = 0; m < d; ++m) rhs[r * 3 + m] -= f * rhs[col * 3 + m];
            }
        }
    }
    for (int r = nb - 1; r >= 0; --r)
        for (int m = 0; m < d; ++m) {
            double s = rhs[r * 3 + m];
            for (int c = r + 1; c < nb; ++c) s -= A[r * 128 + c] * rhs[c * 3 + m];
            rhs[r * 3 + m] = s / A[r * 128 + r];
        }
    for (int t = 0; t < nb; ++t)
        for (int m = 0; m < d; ++m) vel[loc[t] * d + m] = rhs[t * 3 + m];
}

static void damp_visit(int d, double *vel, const int64_t *pi, const int64_t *pj,
                       const double *pd, const double *imi, const double *imj,
                       const int64_t *gp, int64_t g, double half,
                       int64_t *loc, double *A, double *rhs) {
    int64_t lo = gp[g], hi = gp[g + 1];
    if (hi - lo == 1) {
        double c = half * pd[lo];
        damp_pair(d, vel, pi[lo], pj[lo], c * imi[lo], c * imj[lo]);
    } else {
        damp_group(d, vel, pi, pj, pd, imi, imj, half, lo, hi, loc, A, rhs);
    }
}

/* One full sweep: every group forward then reverse, half the step each.
 * `order` (optional, ngroups entries) visits the groups in that sequence
 * instead of 0..ngroups-1 -- used to emulate colour-ordered sweeps. */
void or_damping_sweep(int d, double *vel, const int64_t *pi, const int64_t *pj,
                      const double *pd, const double *imi, const double *imj,
                      int64_t ngroups, const int64_t *gp, const int64_t *order,
                      double eta, double dt) {
    double half = 0.5 * dt * eta;
    int64_t loc[128];
    double *A = (double *)malloc(sizeof(double) * 128 * 128);
    double rhs[128 * 3];
    for (int64_t s = 0; s < ngroups; ++s)
        damp_visit(d, vel, pi, pj, pd, imi, imj, gp, order ? order[s] : s, half, loc, A, rhs);
    for (int64_t s = ngroups - 1; s >= 0; --s)
        damp_visit(d, vel, pi, pj, pd, imi, imj, gp, order ? order[s] : s, half, loc, A, rhs);
    free(A);
}

/* ------------------------------------------------------------ plasticity */

typedef struct {
    double mu, K;              /* shear, bulk */
    double s0, sinf, delta, H; /* law 0: k(a) = s0 + (sinf-s0)(1-e^{-delta a}) + H a
                                  law 1: k(a) = s0 (1 + a/e0)^m with e0 = sinf, m = delta */
    double tol;
    int max_iter;
    int law;
} or_material;

static double hard_k(const or_material *m, double a) {
    if (m->law == 1) return m->s0 * pow(1.0 + a / m->sinf, m->delta);
    return m->s0 + (m->sinf - m->s0) * (1.0 - exp(-m->delta * a)) + m->H * a;
}
static double hard_kp(const or_material *m, double a) {
    if (m->law == 1) return m->s0 * m->delta / m->sinf * pow(1.0 + a / m->sinf, m->delta - 1.0);
    return (m->sinf - m->s0) * m->delta * exp(-m->delta * a) + m->H;
}

/* Return map of one particle (plasticity.py:118).  cp/alpha updated in
 * place.  Returns 0 ok, 1 inverted element, 2 return map failed to
 * converge, 3 plastic tensor inverted.  plastic/dgamma optional outputs. */
static int return_map_one(int d, const double *F, double *cp, double *alpha,
                          const or_material *m, double *tau, double *pk1,
                          int *plastic, double *dgamma, int elastic_only) {
    double j = det_n(d, F);
    if (!(j > 0.0)) return 1;
    double sc = pow(j, -1.0 / d);
    double fb[9], tmp[9], be[9], s[9];
    for (int k = 0; k < d * d; ++k) fb[k] = F[k] * sc;
    if (elastic_only) {
        matmul_nt(d, fb, fb, be);
    } else {
        matmul_n(d, fb, cp, tmp);
        matmul_nt(d, tmp, fb, be);
        for (int r = 0; r < d; ++r)
            for (int c = r + 1; c < d; ++c) {
                double v = 0.5 * (be[r * d + c] + be[c * d + r]);
                be[r * d + c] = v; be[c * d + r] = v;
            }
    }
    double tr = 0.0;
    for (int r = 0; r < d; ++r) tr += be[r * d + r];
    /* s = mu * dev(be) */
    for (int k = 0; k < d * d; ++k) s[k] = m->mu * be[k];
    for (int r = 0; r < d; ++r) s[r * d + r] = m->mu * (be[r * d + r] - tr / d);
    double sn2 = 0.0;
    for (int k = 0; k < d * d; ++k) sn2 += s[k] * s[k];
    double sn = sqrt(sn2);
    int flow = 0;
    double dg = 0.0;
    if (!elastic_only) {
        double fpre = sn - SQ23 * hard_k(m, *alpha);
        flow = fpre > 0.0;
    }
    if (flow) {
        double mue = (tr / d) * m->mu;
        double x = 0.0, lo = 0.0, hi = sn / (2.0 * mue), g = INFINITY;
        for (int it = 0; it < m->max_iter; ++it) {
            double at = *alpha + SQ23 * x;
            g = sn - 2.0 * mue * x - SQ23 * hard_k(m, at);
            if (!(fabs(g) > m->tol)) break;
            if (g > 0.0) lo = x;
            if (g < 0.0) hi = x;
            double gp = -2.0 * mue - (2.0 / 3.0) * hard_kp(m, at);
            double nw = x - g / gp;
            x = (nw > lo && nw < hi) ? nw : 0.5 * (lo + hi);
        }
        g = sn - 2.0 * mue * x - SQ23 * hard_k(m, *alpha + SQ23 * x);
        if (fabs(g) > m->tol) return 2;
        dg = x > 0.0 ? x : 0.0;
        double scale = 1.0 - 2.0 * mue * dg / sn;
        for (int k = 0; k < d * d; ++k) s[k] *= scale;
        *alpha += SQ23 * dg;
        double bn[9], fbi[9];
        for (int k = 0; k < d * d; ++k) bn[k] = s[k] / m->mu;
        for (int r = 0; r < d; ++r) bn[r * d + r] += tr / d;
        inv_n(d, fb, det_n(d, fb), fbi);
        matmul_n(d, fbi, bn, tmp);
        matmul_nt(d, tmp, fbi, cp);
        for (int r = 0; r < d; ++r)
            for (int c = r + 1; c < d; ++c) {
                double v = 0.5 * (cp[r * d + c] + cp[c * d + r]);
                cp[r * d + c] = v; cp[c * d + r] = v;
            }
        double jc = det_n(d, cp);
        if (!(jc > 0.0)) return 3;
        double cs = pow(jc, -1.0 / d);
        for (int k = 0; k < d * d; ++k) cp[k] *= cs;
    }
    double vol = 0.5 * m->K * (j * j - 1.0);
    for (int k = 0; k < d * d; ++k) tau[k] = s[k];
    for (int r = 0; r < d; ++r) tau[r * d + r] += vol;
    double fi[9];
    inv_n(d, F, j, fi);
    matmul_nt(d, tau, fi, pk1);
    if (plastic) *plastic = flow;
    if (dgamma) *dgamma = dg;
    return 0;
}

/* Batched return map.  Returns -1 when all succeed, else the first failing
 * particle id; *status gets the failure kind (1 inversion, 2 no conv). */
int64_t or_return_map(int64_t n, int d, const double *F, double *cp,
                      double *alpha, const double *matp, double *tau,
                      double *pk1, int32_t *plastic, double *dgamma,
                      int elastic_only, int32_t *status) {
    or_material m = {matp[0], matp[1], matp[2], matp[3], matp[4], matp[5],
                     matp[6], (int)matp[7], (int)matp[8]};
    int64_t first = -1;
    int kind = 0;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t a = 0; a < n; ++a) {
        int pl = 0;
        double dg = 0.0;
        int rc = return_map_one(d, F + a * d * d, cp + a * d * d, alpha + a, &m,
                                tau + a * d * d, pk1 + a * d * d, &pl, &dg,
                                elastic_only);
        if (plastic) plastic[a] = pl;
        if (dgamma) dgamma[a] = dg;
        if (rc) {
#pragma omp critical
            { if (first < 0 || a < first) { first = a; kind = rc; } }
        }
    }
    if (status) *status = kind;
    return first;
}

/* --------------------------------------------------- fused necking step */

typedef struct {
    int64_t n;
    int d;
    /* state (reference layout) */
    double *pos, *vel, *F, *accel, *cp, *alpha;
    const double *mass, *rho0;
    const uint8_t *movable;     /* 1 = free */
    const int8_t *side;         /* -1 left clamp, +1 right clamp, 0 other */
    /* neighbourhood */
    const int64_t *indptr, *idx;
    const double *grad0, *vol0, *corr;
    /* damping */
    const int64_t *pi, *pj, *gp, *gorder;
    const double *pd, *imi, *imj;
    int64_t ngroups;
    /* scratch (n*d*d each) */
    double *rate, *pk1, *tmp;
} or_necking;

/* One NeckingProblem.relax_step (scenarios.py:113).  ramp_vbc is the
 * boundary speed when the load ramp is active (ramp_on != 0).  Returns the
 * pre-damping kinetic energy; *err = -1 or the failing particle id. */
double or_necking_relax_step(or_necking *s, double dt, double eta,
                             int ramp_on, double ramp_vbc, const double *matp,
                             int elastic_only, int64_t *err) {
    const int64_t n = s->n;
    const int d = s->d, dd = d * d;
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < n; ++a) {
        if (s->movable[a])
            for (int k = 0; k < d; ++k) s->vel[a * d + k] += 0.5 * dt * s->accel[a * d + k];
        if (ramp_on) {
            if (s->side[a] != 0) {
                for (int k = 0; k < d; ++k) s->vel[a * d + k] = 0.0;
                s->vel[a * d] = s->side[a] < 0 ? -ramp_vbc : ramp_vbc;
            }
        } else if (!s->movable[a]) {
            for (int k = 0; k < d; ++k) s->vel[a * d + k] = 0.0;
        }
        for (int k = 0; k < d; ++k) s->pos[a * d + k] += dt * s->vel[a * d + k];
    }
    or_velocity_gradient_gather(n, d, s->vel, s->indptr, s->idx, s->grad0, s->vol0, s->rate);
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < n; ++a) {
        double r[9];
        matmul_n(d, s->rate + a * dd, s->corr + a * dd, r);
        for (int k = 0; k < dd; ++k) s->F[a * dd + k] += dt * r[k];
    }
    int32_t st = 0;
    *err = or_return_map(n, d, s->F, s->cp, s->alpha, matp, s->tmp, s->pk1, NULL,
                         NULL, elastic_only, &st);
    if (*err >= 0) return NAN;
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < n; ++a) {
        double r[9];
        matmul_n(d, s->pk1 + a * dd, s->corr + a * dd, r);
        memcpy(s->tmp + a * dd, r, sizeof(double) * dd);
    }
    or_pair_tensor_divergence(n, d, s->tmp, s->indptr, s->idx, s->grad0, s->vol0, s->accel);
    double ek = 0.0;
    for (int64_t a = 0; a < n; ++a) {
        for (int k = 0; k < d; ++k) s->accel[a * d + k] /= s->rho0[a];
        if (s->movable[a]) {
            double v2 = 0.0;
            for (int k = 0; k < d; ++k) {
                s->vel[a * d + k] += 0.5 * dt * s->accel[a * d + k];
                v2 += s->vel[a * d + k] * s->vel[a * d + k];
            }
            ek += s->mass[a] * v2;
        }
    }
    ek *= 0.5;
    or_damping_sweep(d, s->vel, s->pi, s->pj, s->pd, s->imi, s->imj, s->ngroups,
                     s->gp, s->gorder, eta, dt);
    return ek;
}

/* solid_time_step (solids.py:187) on the necking state */
double or_necking_stable_dt(const or_necking *s, double h, double c, double cfl) {
    const int d = s->d;
    double vmax2 = 0.0, amax2 = 0.0;
    for (int64_t a = 0; a < s->n; ++a) {
        double v2 = 0.0, a2 = 0.0;
        for (int k = 0; k < d; ++k) {
            v2 += s->vel[a * d + k] * s->vel[a * d + k];
            a2 += s->accel[a * d + k] * s->accel[a * d + k];
        }
        if (v2 > vmax2) vmax2 = v2;
        if (s->movable[a] && a2 > amax2) amax2 = a2;
    }
    double dt = h / (c + sqrt(vmax2));
    double amax = sqrt(amax2);
    if (amax > 0.0) { double t = sqrt(h / amax); if (t < dt) dt = t; }
    return cfl * dt;
}

int or_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* thread count of the parallel loops (the reference arm of bench.py runs
   under torchrun, which exports OMP_NUM_THREADS=1) */
void or_set_num_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
