// solid.cuh -- total-Lagrangian elastoplastic inner relaxation on the GPU.
//
// One inner step = NeckingProblem.relax_step (scenarios.py:113) + the
// stepping.py:158 bookkeeping, as five kernels plus the damping sweep:
//
//   k_solid_kick_drift : v += dt/2 a (free), boundary ramp / clamps, x += dt v
//   k_solid_stress     : SELL gather dF/dt = (sum_b V_b (v_b - v_a) (x) gradW) B
//                        (solids.py:118), F += dt dF/dt, J2 return map or
//                        Neo-Hookean stress (plasticity.py:118, solids.py:148),
//                        T = P B stored for the divergence
//   k_solid_accel      : SELL gather a = 1/rho0 sum_b V_b (T_a + T_b) gradW
//                        (solids.py:170), v += dt/2 a, E_k and |a|max partials
//   sweep              : damping (damping.cuh)
//   k_solid_vmax       : |v|max partial after damping
//   k_solid_ctrl       : 1 block: fixed-order reductions, convergence test,
//                        counters, next dt (solids.py:187) -- all on device
//
// State lives in HBM in the Morton order of the neighbourhood: own-access
// fields SoA (coalesced), gathered fields AoS (X|vol and v as one 32 B
// sector, T planar 72 B -- see TS below), so a neighbour costs whole sectors.
#pragma once

#include "damping.cuh"
#include "nbh.cuh"

namespace mtsph {

// FL_GHOST: a halo copy of another rank's particle (multi-GPU); its state
// is written by exchanges only and it is excluded from every reduction
enum { FL_MOVABLE = 1, FL_LEFT = 2, FL_RIGHT = 4, FL_MID = 8, FL_GHOST = 16 };

struct Mat {
    double mu, K;
    double p[4];   // law 0: s0, sinf, delta, H ; law 1: s0, e0, m, -
    double tol;
    int max_iter;
    int law;
    int plastic;
};

// t^m for t >= 1 (the power law's 1 + a/e0): exp2(m log2 t) is within a
// few 1e-17 of pow here (m log2 t is small) and cheaper than pow's
// extra-precise path
__device__ __forceinline__ double pow_ge1(double t, double m) { return exp2(m * log2(t)); }

// LAW: the hardening law as a compile-time constant (0, 1), or -1 to
// read m.law at run time.  The split return-map kernels are instantiated
// per law, so each carries one law's code and registers.
template <int LAW = -1> __device__ __forceinline__ double hard_k(const Mat &m, double a) {
    if (LAW == 1 || (LAW < 0 && m.law == 1)) return m.p[0] * pow_ge1(1.0 + a / m.p[1], m.p[2]);
    return m.p[0] + (m.p[1] - m.p[0]) * (1.0 - exp(-m.p[2] * a)) + m.p[3] * a;
}
// K(a) and K'(a) from one pow / exp (the Newton iterate needs both):
// law 1: K' = m K / (e0 (1 + a/e0)), equal to s0 m/e0 (1 + a/e0)^(m-1) up
// to rounding; law 0: K' = (sinf - s0) delta e^(-delta a) + H
template <int LAW = -1> __device__ __forceinline__ double hard_k_kp(const Mat &m, double a, double &kp) {
    if (LAW == 1 || (LAW < 0 && m.law == 1)) {
        const double t = 1.0 + a / m.p[1];
        const double k = m.p[0] * pow_ge1(t, m.p[2]);
        kp = k * m.p[2] / (m.p[1] * t);
        return k;
    }
    const double e = exp(-m.p[2] * a);
    kp = (m.p[1] - m.p[0]) * m.p[2] * e + m.p[3];
    return m.p[0] + (m.p[1] - m.p[0]) * (1.0 - e) + m.p[3] * a;
}

#define SQ23_D 0.81649658092772603273

// plasticity.py:118 for one particle.  Returns 0, 1 (det F <= 0),
// 2 (no convergence), 3 (plastic tensor inverted).
template <int D, int LAW = -1>
__device__ __forceinline__ int return_map_dev(const double *F, double *cp, double &alpha, const Mat &m,
                                              double *P) {
    const double j = det_d<D>(F);
    if (!(j > 0.0)) return 1;
    const double sc = det_pow_minus_inv_d<D>(j);
    double fb[D * D], be[D * D], s[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) fb[k] = F[k] * sc;
    if (m.plastic) {
        double tmp[D * D];
        mm<D>(fb, cp, tmp);
        mmt<D>(tmp, fb, be);
#pragma unroll
        for (int r = 0; r < D; ++r)
#pragma unroll
            for (int c = r + 1; c < D; ++c) {
                const double v = 0.5 * (be[r * D + c] + be[c * D + r]);
                be[r * D + c] = v;
                be[c * D + r] = v;
            }
    } else {
        mmt<D>(fb, fb, be);
    }
    double tr = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) tr += be[r * D + r];
#pragma unroll
    for (int k = 0; k < D * D; ++k) s[k] = m.mu * be[k];
#pragma unroll
    for (int r = 0; r < D; ++r) s[r * D + r] = m.mu * (be[r * D + r] - tr / D);
    if (m.plastic) {
        double sn2 = 0.0;
#pragma unroll
        for (int k = 0; k < D * D; ++k) sn2 += s[k] * s[k];
        const double sn = sqrt(sn2);
        double kp;
        double kat = hard_k_kp<LAW>(m, alpha, kp);   // K, K' at the first iterate (x = 0)
        const double fpre = sn - SQ23_D * kat;
        if (fpre > 0.0) {
            const double mue = (tr / D) * m.mu;
            // plasticity.py:118 Newton-bisection.  One hardening evaluation
            // per iterate (the first is the trial-state one above); when the
            // loop stops on the tolerance the residual of the final x is the
            // one just computed (same x), so only an exhausted loop
            // re-evaluates it.
            double x = 0.0, lo = 0.0, hi = sn / (2.0 * mue), gf = 0.0;
            bool conv = false;
            for (int it = 0; it < m.max_iter; ++it) {
                if (it > 0) kat = hard_k_kp<LAW>(m, alpha + SQ23_D * x, kp);
                const double g = sn - 2.0 * mue * x - SQ23_D * kat;
                if (!(fabs(g) > m.tol)) { gf = g; conv = true; break; }
                if (g > 0.0) lo = x;
                if (g < 0.0) hi = x;
                const double gp = -2.0 * mue - (2.0 / 3.0) * kp;
                const double nw = x - g / gp;
                x = (nw > lo && nw < hi) ? nw : 0.5 * (lo + hi);
            }
            if (!conv) gf = sn - 2.0 * mue * x - SQ23_D * hard_k<LAW>(m, alpha + SQ23_D * x);
            if (fabs(gf) > m.tol) return 2;
            const double dg = x > 0.0 ? x : 0.0;
            const double scale = 1.0 - 2.0 * mue * dg / sn;
#pragma unroll
            for (int k = 0; k < D * D; ++k) s[k] *= scale;
            alpha += SQ23_D * dg;
            double bn[D * D], fbi[D * D], tmp[D * D];
#pragma unroll
            for (int k = 0; k < D * D; ++k) bn[k] = s[k] / m.mu;
#pragma unroll
            for (int r = 0; r < D; ++r) bn[r * D + r] += tr / D;
            inv_d<D>(fb, det_d<D>(fb), fbi);
            mm<D>(fbi, bn, tmp);
            mmt<D>(tmp, fbi, cp);
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
                for (int c = r + 1; c < D; ++c) {
                    const double v = 0.5 * (cp[r * D + c] + cp[c * D + r]);
                    cp[r * D + c] = v;
                    cp[c * D + r] = v;
                }
            const double jc = det_d<D>(cp);
            if (!(jc > 0.0)) return 3;
            const double cs = det_pow_minus_inv_d<D>(jc);
#pragma unroll
            for (int k = 0; k < D * D; ++k) cp[k] *= cs;
        }
    }
    const double vol = 0.5 * m.K * (j * j - 1.0);
#pragma unroll
    for (int r = 0; r < D; ++r) s[r * D + r] += vol;
    double fi[D * D];
    inv_d<D>(F, j, fi);
    mmt<D>(s, fi, P);
    return 0;
}

// Divergence tensor T = P B^T, gathered once per neighbour by the
// acceleration kernel.  2D: one double4 per particle.  3D: planar, 72 B per
// particle with no padding -- plane 0 = double4 (T00 T01 T02 T10), plane 1 =
// double4 (T11 T12 T20 T21), plane 2 = double (T22) -- so the gather fetches
// 9 doubles instead of three padded 32 B rows, and consecutive particles
// share the sectors of the scalar plane.
template <int D> struct TS { static constexpr int n = D == 3 ? 9 : 4; };

// (tload: only from kernels that do not write T -- non-coherent loads)
template <int D> __device__ __forceinline__ void tload(const double *Tp, int64_t n, int64_t a, double *t) {
    const double4 *r = reinterpret_cast<const double4 *>(Tp);
    if (D == 2) {
        const double4 q = ldg4(r + a);
        t[0] = q.x; t[1] = q.y; t[2] = q.z; t[3] = q.w;
    } else {
        const double4 q0 = ldg4(r + a), q1 = ldg4(r + n + a);
        t[0] = q0.x; t[1] = q0.y; t[2] = q0.z; t[3] = q0.w;
        t[4] = q1.x; t[5] = q1.y; t[6] = q1.z; t[7] = q1.w;
        t[8] = __ldg(Tp + 8 * n + a);
    }
}
template <int D> __device__ __forceinline__ void tstore(double *Tp, int64_t n, int64_t a, const double *t) {
    double4 *r = reinterpret_cast<double4 *>(Tp);
    if (D == 2) {
        st4(r + a, make_double4(t[0], t[1], t[2], t[3]));
    } else {
        st4(r + a, make_double4(t[0], t[1], t[2], t[3]));
        st4(r + n + a, make_double4(t[4], t[5], t[6], t[7]));
        Tp[8 * n + a] = t[8];
    }
}

// Solid divergence record: T~ = V0 T (the neighbour's volume folded in) and,
// in 3D, the reference position in the same three 32 B planes, so the
// acceleration gather reads three 256-bit records per neighbour and nothing
// else (sum_b V_b gradW, the T_a part, is static: SolidArgs::G).
//   3D: (T~00 T~01 T~02 T~10) (T~11 T~12 T~20 T~21) (X0 X1 X2 T~22)
//   2D: (T~00 T~01 T~10 T~11), X from XV
template <int D> struct DS { static constexpr int n = D == 3 ? 12 : 4; };

// store T~ (already scaled) with the particle's reference position
template <int D>
__device__ __forceinline__ void dstore_raw(double *Tp, int64_t n, int64_t a, const double *tt, const double4 &xv) {
    double4 *r = reinterpret_cast<double4 *>(Tp);
    if (D == 2) {
        st4(r + a, make_double4(tt[0], tt[1], tt[2], tt[3]));
    } else {
        st4(r + a, make_double4(tt[0], tt[1], tt[2], tt[3]));
        st4(r + n + a, make_double4(tt[4], tt[5], tt[6], tt[7]));
        st4(r + 2 * n + a, make_double4(xv.x, xv.y, xv.z, tt[8]));
    }
}
// (read-only kernels) T~ and the reference position of particle b
template <int D>
__device__ __forceinline__ void dload(const double *Tp, int64_t n, const double4 *XV, int64_t b, double *tt,
                                      double *x) {
    const double4 *r = reinterpret_cast<const double4 *>(Tp);
    const double4 q0 = ldg4(r + b);
    if (D == 2) {
        tt[0] = q0.x; tt[1] = q0.y; tt[2] = q0.z; tt[3] = q0.w;
        const double4 xv = ldg4(XV + b);
        x[0] = xv.x; x[1] = xv.y;
    } else {
        const double4 q1 = ldg4(r + n + b), q2 = ldg4(r + 2 * n + b);
        tt[0] = q0.x; tt[1] = q0.y; tt[2] = q0.z; tt[3] = q0.w;
        tt[4] = q1.x; tt[5] = q1.y; tt[6] = q1.z; tt[7] = q1.w;
        tt[8] = q2.w;
        x[0] = q2.x; x[1] = q2.y; x[2] = q2.z;
    }
}

struct SolidArgs {
    int64_t n;
    const double4 *XV;
    void *V;
    double *x, *a, *F, *cp, *alpha, *T;   // T: divergence records (DS)
    const double *B, *mass, *rho0;
    const double *G;         // [d][n] sum_b V_b gradW_ab (static, setup)
    const uint8_t *flags;
    const int64_t *slice_ptr;
    const int32_t *slice_w, *nbr;
    const int64_t *indptr;   // CSR rows (sorted), for the row-parallel gathers
    const int32_t *csr;
    const int64_t *cptr;     // chunked index table (gather_csr.cuh): chunk offsets, or null
    const int32_t *csr16;
    const double *mag16;     // per entry of csr16: kernel-gradient magnitude factor, or null
    const int64_t *perm;
    const double *Lacc;  // window gathers: sum_b V_b (v_b-v_a) (x) gradW [d*d][n] (F updated in k_solid_rmap)
    double *part;    // [3][nblk]: ek, amax2, vmax2
    int nblk;
    Ctrl *ctrl;
    KSpec ks;
    Mat mat;
};

// return map + T = P B for one particle (shared by the fused and split paths)
template <int D, int LAW = -1>
__device__ __forceinline__ void solid_stress_point(const SolidArgs &A, int64_t i, const double *F,
                                                          const double *Bm) {
    const int64_t n = A.n;
    Ctrl *c = A.ctrl;
    double cp[D * D];
    double alpha = 0.0;
    if (A.mat.plastic) {
#pragma unroll
        for (int k = 0; k < D * D; ++k) cp[k] = A.cp[(int64_t)k * n + i];
        alpha = A.alpha[i];
    }
    double P[D * D];
    const int rc = return_map_dev<D, LAW>(F, cp, alpha, A.mat, P);
    if (rc) {
        const unsigned long long id = (unsigned long long)A.perm[i];
        if (rc == 1) atomicMin(&c->err_inv, id);
        else atomicMin(&c->err_rm, id);
#pragma unroll
        for (int k = 0; k < D * D; ++k) P[k] = 0.0;
    } else if (A.mat.plastic) {
#pragma unroll
        for (int k = 0; k < D * D; ++k) A.cp[(int64_t)k * n + i] = cp[k];
        A.alpha[i] = alpha;
    }
    double Tm[D * D];
    if (Bm) {
        mm<D>(P, Bm, Tm);
    } else {  // B read only now: not live across the return map (registers)
        double Bl[D * D];
#pragma unroll
        for (int k = 0; k < D * D; ++k) Bl[k] = A.B[(int64_t)k * n + i];
        mm<D>(P, Bl, Tm);
    }
    const double4 xv = ldg4(A.XV + i);
    const double vol = volof<D>(xv);
#pragma unroll
    for (int k = 0; k < D * D; ++k) Tm[k] *= vol;
    dstore_raw<D>(A.T, A.n, i, Tm, xv);
}

// sum_b V_b gradW_ab per particle, CSR row order (static; once at setup)
template <int D>
__global__ void __launch_bounds__(256) k_solid_gsum(SolidArgs A, double *G) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    double xa[3], s[D];
    xget<D>(ldg4(A.XV + i), xa);
#pragma unroll
    for (int k = 0; k < D; ++k) s[k] = 0.0;
    for (int64_t k = A.indptr[i]; k < A.indptr[i + 1]; ++k) {
        const double4 xvb = ldg4(A.XV + A.csr[k]);
        double xb[3], rel[D], g[D];
        xget<D>(xvb, xb);
#pragma unroll
        for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
        grad_w<D>(rel, A.ks, g);
        const double volb = volof<D>(xvb);
#pragma unroll
        for (int q = 0; q < D; ++q) s[q] += volb * g[q];
    }
#pragma unroll
    for (int k = 0; k < D; ++k) G[(int64_t)k * A.n + i] = s[k];
}

template <int D>
__global__ void __launch_bounds__(256) k_solid_kick_drift(SolidArgs A) {
    using V_t = typename VT<D>::T;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const double dt = c->dt;
    const uint8_t f = A.flags[i];
    if (f & FL_GHOST) return;  // another rank integrates it
    V_t *V = reinterpret_cast<V_t *>(A.V);
    double v[3];
    vget(V[i], v);
    if (f & FL_MOVABLE) {
#pragma unroll
        for (int k = 0; k < D; ++k) v[k] += 0.5 * dt * A.a[(int64_t)k * A.n + i];
    }
    if (c->ramp_left > 0) {
        if (f & (FL_LEFT | FL_RIGHT)) {
            const double vbc = c->ramp_disp / dt;
#pragma unroll
            for (int k = 0; k < D; ++k) v[k] = 0.0;
            v[0] = (f & FL_LEFT) ? -vbc : vbc;
        }
    } else if (!(f & FL_MOVABLE)) {
#pragma unroll
        for (int k = 0; k < D; ++k) v[k] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) A.x[(int64_t)k * A.n + i] += dt * v[k];
    V_t w;
    vset(w, v);
    V[i] = w;
}


template <int D, bool SPLIT>
__global__ void __launch_bounds__(256) k_solid_stress(SolidArgs A) {
    using V_t = typename VT<D>::T;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    Ctrl *c = A.ctrl;
    if (c->done) return;
    if (A.flags[i] & FL_GHOST) return;
    const double dt = c->dt;
    const int64_t n = A.n;
    const V_t *V = reinterpret_cast<const V_t *>(A.V);
    double xa[3], va[3];
    xget<D>(ldg4(A.XV + i), xa);
    vget(vldg(V + i), va);
    double acc[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) acc[k] = 0.0;
    const int64_t s = i >> 5;
    const int lane = (int)(i & 31);
    const int64_t base = A.slice_ptr[s] + lane;
    const int w = A.slice_w[s];
    for (int m = 0; m < w; ++m) {
        const int32_t b = __ldg(A.nbr + base + (int64_t)m * 32);
        const double4 xvb = ldg4(A.XV + b);
        double xb[3], vb[3], rel[D], g[D];
        xget<D>(xvb, xb);
        vget(vldg(V + b), vb);
#pragma unroll
        for (int k = 0; k < D; ++k) rel[k] = xb[k] - xa[k];
        grad_w<D>(rel, A.ks, g);
        const double volb = volof<D>(xvb);
#pragma unroll
        for (int r = 0; r < D; ++r) {
            const double dv = volb * (vb[r] - va[r]);
#pragma unroll
            for (int cc = 0; cc < D; ++cc) acc[r * D + cc] += dv * g[cc];
        }
    }
    double Bm[D * D], F[D * D], L[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) {
        Bm[k] = A.B[(int64_t)k * n + i];
        F[k] = A.F[(int64_t)k * n + i];
    }
    mm<D>(acc, Bm, L);
#pragma unroll
    for (int k = 0; k < D * D; ++k) F[k] += dt * L[k];
#pragma unroll
    for (int k = 0; k < D * D; ++k) A.F[(int64_t)k * n + i] = F[k];
    if (SPLIT) return;
    solid_stress_point<D>(A, i, F, Bm);
}

// element-wise second half of the split stress kernel: return map + T
template <int D, int LAW>
__global__ void __launch_bounds__(256, 2) k_solid_rmap(SolidArgs A) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    if (A.ctrl->done) return;
    if (A.flags[i] & FL_GHOST) return;
    const int64_t n = A.n;
    double F[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) F[k] = A.F[(int64_t)k * n + i];
    if (A.Lacc) {  // after a window gather: F += dt (sum) B, as the CSR gather's epilogue
        const double dt = A.ctrl->dt;
        double acc[D * D], Bm[D * D], L[D * D];
#pragma unroll
        for (int k = 0; k < D * D; ++k) {
            acc[k] = A.Lacc[(int64_t)k * n + i];
            Bm[k] = A.B[(int64_t)k * n + i];
        }
        mm<D>(acc, Bm, L);
#pragma unroll
        for (int k = 0; k < D * D; ++k) {
            F[k] = F[k] + dt * L[k];
            A.F[(int64_t)k * n + i] = F[k];
        }
    }
    solid_stress_point<D, LAW>(A, i, F, nullptr);
}

template <int D>
__global__ void __launch_bounds__(256) k_solid_accel(SolidArgs A) {
    using V_t = typename VT<D>::T;
    __shared__ double sh[32];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const Ctrl *c = A.ctrl;
    if (c->done) return;  // uniform across the grid
    double ek = 0.0, a2m = 0.0;
    if (i < A.n && !(A.flags[i] & FL_GHOST)) {
        const double dt = c->dt;
        const double4 xva = ldg4(A.XV + i);
        double xa[3];
        xget<D>(xva, xa);
        double acc[D];
#pragma unroll
        for (int k = 0; k < D; ++k) acc[k] = 0.0;
        const int64_t s = i >> 5;
        const int lane = (int)(i & 31);
        const int64_t base = A.slice_ptr[s] + lane;
        const int w = A.slice_w[s];
        for (int m = 0; m < w; ++m) {
            const int32_t b = __ldg(A.nbr + base + (int64_t)m * 32);
            double xb[3], Tb[D * D], rel[D], g[D];
            dload<D>(A.T, A.n, A.XV, b, Tb, xb);
#pragma unroll
            for (int k = 0; k < D; ++k) rel[k] = xb[k] - xa[k];
            grad_w<D>(rel, A.ks, g);
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double sum = 0.0;
#pragma unroll
                for (int cc = 0; cc < D; ++cc) sum += Tb[r * D + cc] * g[cc];
                acc[r] += sum;
            }
        }
        // + T_a sum_b V_b gradW = (T~_a / V_a) G_a
        double Ta[D * D], xd[3];
        dload<D>(A.T, A.n, A.XV, i, Ta, xd);
        const double rho0 = A.rho0[i], vola = volof<D>(xva);
#pragma unroll
        for (int k = 0; k < D; ++k) {
            double ta = 0.0;
#pragma unroll
            for (int cc = 0; cc < D; ++cc) ta += Ta[k * D + cc] * A.G[(int64_t)cc * A.n + i];
            acc[k] = (acc[k] + ta / vola) / rho0;
            A.a[(int64_t)k * A.n + i] = acc[k];
        }
        if (A.flags[i] & FL_MOVABLE) {
            V_t *V = reinterpret_cast<V_t *>(A.V);
            double v[3];
            vget(V[i], v);
            double v2 = 0.0, aa = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                v[k] += 0.5 * dt * acc[k];
                v2 += v[k] * v[k];
                aa += acc[k] * acc[k];
            }
            V_t w2;
            vset(w2, v);
            V[i] = w2;
            ek = A.mass[i] * v2;
            a2m = aa;
        }
    }
    const double se = block_sum<256>(ek, sh);
    const double sa = block_max<256>(a2m, sh);
    if (threadIdx.x == 0) {
        A.part[blockIdx.x] = se;
        A.part[A.nblk + blockIdx.x] = sa;
    }
}


// |v|^2 max over all particles (mode 0) or also |a|^2 over the free ones
// (mode 1, used before the first step)
template <int D>
__global__ void __launch_bounds__(256) k_solid_vmax(SolidArgs A, int with_accel) {
    using V_t = typename VT<D>::T;
    __shared__ double sh[32];
    if (!with_accel && A.ctrl->done) return;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double v2 = 0.0, a2 = 0.0;
    if (i < A.n && !(A.flags[i] & FL_GHOST)) {
        const V_t *V = reinterpret_cast<const V_t *>(A.V);
        double v[3];
        vget(V[i], v);
#pragma unroll
        for (int k = 0; k < D; ++k) v2 += v[k] * v[k];
        if (with_accel && (A.flags[i] & FL_MOVABLE)) {
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const double q = A.a[(int64_t)k * A.n + i];
                a2 += q * q;
            }
        }
    }
    const double mv = block_max<256>(v2, sh);
    const double ma = block_max<256>(a2, sh);
    if (threadIdx.x == 0) {
        A.part[2 * A.nblk + blockIdx.x] = mv;
        if (with_accel) A.part[A.nblk + blockIdx.x] = ma;
    }
}

enum { CTRL_INIT = 0, CTRL_STEP = 1, CTRL_SINGLE = 2 };

__device__ __forceinline__ double stable_dt(const Ctrl *c, double vmax2, double amax2) {
    double dt = c->h / (c->sound + sqrt(vmax2));
    const double amax = sqrt(amax2);
    if (amax > 0.0) dt = fmin(dt, sqrt(c->h / amax));
    return c->cfl * dt;
}

// the stopping rule and next step from the reduced E_k sum, |a|max^2 and
// |v|max^2 (stepping.py:177-195, solids.py:187); one thread
__device__ __forceinline__ void ctrl_apply(Ctrl *c, double E, double AM, double VM, int mode) {
    c->amax2 = AM;
    c->vmax2 = VM;
    if (mode == CTRL_INIT) {
        c->dt = stable_dt(c, VM, AM);
        return;
    }
    const double ek = 0.5 * E * (c->vol_movable > 0.0 ? 1.0 / c->vol_movable : 1.0);
    c->ek = ek;
    if (c->ramp_left > 0) c->ramp_left -= 1;
    if (c->err_inv != ~0ull || c->err_rm != ~0ull) { c->done = 1; return; }
    if (mode == CTRL_SINGLE) return;
    const double dt_used = c->dt;
    c->n_inner += 1;
    c->last_dt = dt_used;
    c->min_dt = fmin(c->min_dt, dt_used);
    const bool conv = ek <= c->criterion;
    long long cap = c->max_inner;
    if (cap <= 0) cap = 10 * (long long)ceil(c->dt_outer / dt_used);
    if (conv && c->n_inner >= c->min_inner && c->ramp_left <= 0) { c->done = 1; return; }
    if (c->n_inner >= cap) { c->done = 1; c->cap_hit = 1; return; }
    c->dt = stable_dt(c, VM, AM);
}

// one block of kCtrlThreads; fixed-order reduction of the per-block partials
constexpr int kCtrlThreads = 1024;
__global__ void __launch_bounds__(kCtrlThreads) k_ctrl(Ctrl *c, const double *part, int nblk, int mode) {
    __shared__ double sh[32];
    if (mode == CTRL_STEP && c->done) return;
    double e = 0.0, am = 0.0, vm = 0.0;
    for (int b = threadIdx.x; b < nblk; b += kCtrlThreads) {
        if (mode != CTRL_INIT) e += part[b];
        am = fmax(am, part[nblk + b]);
        vm = fmax(vm, part[2 * nblk + b]);
    }
    const double E = block_sum<kCtrlThreads>(e, sh);
    const double AM = block_max<kCtrlThreads>(am, sh);
    const double VM = block_max<kCtrlThreads>(vm, sh);
    if (threadIdx.x == 0) ctrl_apply(c, E, AM, VM, mode);
}

// Multi-rank device control.  k_rank_partials reduces this rank's
// per-block partials (owned particles only) to out[4] = {sum m v^2,
// max |a|^2, max |v|^2, error flag}; the ranks' quadruples are all-gathered
// (NCCL) into [nranks][4] and k_ctrl_ranks reduces them in rank order -- the same
// operations on every rank, so all ranks take identical control decisions
// without the host.
__global__ void __launch_bounds__(256) k_rank_partials(const Ctrl *c, const double *part, int nblk, int mode,
                                                       double *out) {
    __shared__ double sh[32];
    if (mode == CTRL_STEP && c->done) return;
    double e = 0.0, am = 0.0, vm = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 256) {
        if (mode != CTRL_INIT) e += part[b];
        am = fmax(am, part[nblk + b]);
        vm = fmax(vm, part[2 * nblk + b]);
    }
    const double E = block_sum<256>(e, sh);
    const double AM = block_max<256>(am, sh);
    const double VM = block_max<256>(vm, sh);
    if (threadIdx.x == 0) {
        out[0] = E;
        out[1] = AM;
        out[2] = VM;
        out[3] = (c->err_inv != ~0ull || c->err_rm != ~0ull) ? 1.0 : 0.0;
    }
}

// gathered: [nranks][4] = {sum m v^2, max |a|^2, max |v|^2, error flag};
// an error on any rank stops every rank
__global__ void k_ctrl_ranks(Ctrl *c, const double *gathered, int nranks, int mode) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (mode == CTRL_STEP && c->done) return;
    double E = 0.0, AM = 0.0, VM = 0.0, err = 0.0;
    for (int r = 0; r < nranks; ++r) {
        E += gathered[4 * r];
        AM = fmax(AM, gathered[4 * r + 1]);
        VM = fmax(VM, gathered[4 * r + 2]);
        err = fmax(err, gathered[4 * r + 3]);
    }
    ctrl_apply(c, E, AM, VM, mode);
    if (err > 0.0) {
        c->done = 1;
        // a rank without an error of its own still has to fail (its host
        // would otherwise enter the next outer step's exchanges alone)
        if (c->err_inv == ~0ull && c->err_rm == ~0ull) c->remote_err = 1;
    }
}

// observables (NeckingProblem.measure) as per-block partials
template <int D>
__global__ void __launch_bounds__(256) k_solid_measure(SolidArgs A, double *out /* [5][nblk] */) {
    using V_t = typename VT<D>::T;
    __shared__ double sh[32];
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double fx = 0.0, rad = 0.0, amax = 0.0, amin = 1e308, bad = 0.0;
    if (i < A.n && !(A.flags[i] & FL_GHOST)) {
        const uint8_t f = A.flags[i];
        if (f & FL_RIGHT) fx = A.mass[i] * A.a[i];
        if (f & FL_MID) {
            double r2 = 0.0;
#pragma unroll
            for (int k = 1; k < D; ++k) {
                const double q = A.x[(int64_t)k * A.n + i];
                r2 += q * q;
            }
            rad = sqrt(r2);
            if (A.mat.plastic) amin = A.alpha[i];
        }
        if (A.mat.plastic) amax = A.alpha[i];
        double v[3];
        vget(reinterpret_cast<const V_t *>(A.V)[i], v);
#pragma unroll
        for (int k = 0; k < D; ++k) if (!isfinite(v[k])) bad = 1.0;
    }
    const double s0 = block_sum<256>(fx, sh);
    const double s1 = block_max<256>(rad, sh);
    const double s2 = block_max<256>(amax, sh);
    const double s3 = block_min<256>(amin, sh);
    const double s4 = block_max<256>(bad, sh);
    if (threadIdx.x == 0) {
        const int nb = gridDim.x;
        out[blockIdx.x] = s0;
        out[nb + blockIdx.x] = s1;
        out[2 * nb + blockIdx.x] = s2;
        out[3 * nb + blockIdx.x] = s3;
        out[4 * nb + blockIdx.x] = s4;
    }
}

}  // namespace mtsph
