// porous.cuh -- partially saturated porous membrane on the GPU.
//
// Outer (slow) step = PorousProblem.advance_slow (scenarios.py:226):
//   k_por_prep      J, current volume, rho_l, saturation, D rho_l, and the
//                   gradient map A = F^-1 B^T              (porous.py:133-139)
//   k_por_flux      q_a = D rho_l,a sum_b V_b (s_a - s_b) (A_a gradW)    (:503)
//   k_por_mass      conservative pair-form mass rate, gathered per
//                   particle (no atomics, fixed order), clamp + counting,
//                   contact constraint / evaporation                      (:476)
//   k_por_post      pressure, mixture masses, momentum rebuild, solid /
//                   fluid velocity split with the dry guard               (:601)
//   k_por_fluxrate  advected-momentum rate -sum V_b (vq_a+vq_b).(A_a gradW) (:574)
// Inner step = PorousProblem.relax_step (scenarios.py:278):
//   k_por_kick1     M += dt/2 rate, clamps, v_s, x += dt v_s
//   k_por_stress    gather dF/dt, F += dt dF/dt                        (_accel.py:240)
//   k_por_constit   J, Almansi mixture stress, nominal stress, divergence
//                   record T~ = V0 Pm B (solid.cuh DS layout, X included)
//   k_por_accel     gather of sum_b T~_b.gradW + T_a sum_b V_b gradW
//                   (static, G) + flux rate, kick,
//                   energy-density / |a| partials
//   sweep           damping with mixture masses
//   k_por_post_step momentum rebuild, |v|max partial
//
// Every neighbour gather is row-parallel (gather_csr.cuh): kPorLanes lanes
// per particle walk its sorted CSR row with stride kPorLanes, the partial
// sums are combined by a fixed xor-shuffle tree, and lane 0 of the group
// runs the particle's epilogue.  A block covers 256 particles in kPorLanes
// rounds, so grids and per-block partials are those of one thread per
// particle.
#pragma once

#include "damping.cuh"
#include "gather_csr.cuh"
#include "solid.cuh"

namespace mtsph {

// PF_GHOST: a halo copy of another rank's particle (multi-rank): never
// updated here (its fields come from exchanges), never reduced
enum { PF_MOVABLE = 1, PF_CONTACT = 2, PF_GHOST = 4 };

struct PorMat {
    double rho_s0, D, C, mu, lam, porosity, rho_l0, sat0;
};

struct PorousArgs {
    int64_t n;
    const double4 *XV;
    void *V;                        // solid velocity (VT<D>)
    double *x, *F, *M, *q, *vl, *rate, *frate;
    double *mass_l, *sat, *pres, *J, *rho_lf, *mix, *inv_mix;
    double *volc, *coeff, *amap, *mrate;
    double *T;                      // divergence records (DS<D>)
    // planar gather records of the outer step: plane k of particle b is the
    // 32 B at (k n + b), so the 4 lanes of a row group (4 consecutive
    // neighbours) read one 128 B line per plane instead of one sector per
    // scalar field.  rm (mass update): 3D (A00 A01 A02 A10) (A11 A12 A20 A21)
    // (A22 q0 q1 q2) (X0 X1 X2 V); 2D (A00 A01 A10 A11) (q0 q1 V 0), X from
    // XV.  rf (flux rate): (vl0 vl1 vl2|0 V) (q0 q1 q2|0 0), X from XV.
    double *rm, *rf;
    const double *G;                // [d][n] sum_b V_b gradW_ab (static)
    const double *B;
    const uint8_t *flags;
    const int64_t *indptr;   // CSR rows (sorted)
    const int64_t *cptr;     // chunked index table (gather_csr.cuh build_chunked, kPorLanes lanes)
    const int32_t *csr16;
    const double *mag16;     // stored kernel-gradient magnitude factors per entry of csr16
    const int32_t *csr;
    const int64_t *perm;
    double *part;
    int nblk;
    Ctrl *ctrl;
    KSpec ks;
    PorMat m;
};

constexpr int kPorLanes = 4;
// dF/dt gather from the stored gradient magnitudes (1) or recomputed (0)
#ifndef MTSPH_POR_STRESS_MAG
#define MTSPH_POR_STRESS_MAG 1
#endif
template <int D> struct PorRM { static constexpr int planes = D == 3 ? 4 : 2; };

// particle of round `it` for this lane, its lane within the group
#define POR_ROWS_BEGIN                                                              \
    const int sub = threadIdx.x % kPorLanes;                                         \
    for (int it = 0; it < kPorLanes; ++it) {                                         \
        const int64_t i = (int64_t)blockIdx.x * 256 + it * (256 / kPorLanes) + threadIdx.x / kPorLanes; \
        const bool act = i < n;
#define POR_ROWS_END }

// this lane's neighbours of particle i from the chunked index table (gather_csr.cuh)
template <bool FAST = true, class F>
__device__ __forceinline__ void por_walk(const PorousArgs &A, int64_t i, int sub, F &&visit) {
    walk_chunks_any<kPorLanes, FAST ? 2 : 0, false>(A.cptr, A.csr16, nullptr, i, sub, visit);
}
// the same with the stored gradient magnitudes: visit(b, mag)
template <bool FAST = true, class F>
__device__ __forceinline__ void por_walk_mag(const PorousArgs &A, int64_t i, int sub, F &&visit) {
    walk_chunks_any<kPorLanes, FAST ? 2 : 0, true>(A.cptr, A.csr16, A.mag16, i, sub, visit);
}

template <int D>
__global__ void __launch_bounds__(256) k_por_prep(PorousArgs A, int with_amap) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    if (A.flags[i] & PF_GHOST) return;
    const int64_t n = A.n;
    double F[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) F[k] = A.F[(int64_t)k * n + i];
    const double j = det_d<D>(F);
    if (!(j > 0.0)) atomicMin(&A.ctrl->err_inv, (unsigned long long)A.perm[i]);
    const double vol = volof<D>(A.XV[i]) * j;
    const double rho_l = A.mass_l[i] / vol;
    A.volc[i] = vol;
    A.sat[i] = rho_l / A.m.rho_l0;
    A.coeff[i] = A.m.D * rho_l;
    A.J[i] = j;
    if (with_amap) {
        double fi[D * D], Bm[D * D], am[D * D];
        inv_d<D>(F, j, fi);
#pragma unroll
        for (int k = 0; k < D * D; ++k) Bm[k] = A.B[(int64_t)k * n + i];
        mmt<D>(fi, Bm, am);  // F^-1 B^T
#pragma unroll
        for (int k = 0; k < D * D; ++k) A.amap[(int64_t)k * n + i] = am[k];
        double4 *rm = reinterpret_cast<double4 *>(A.rm);
        if (D == 3) {
            const double4 xv = ldg4(A.XV + i);
            st4(rm + i, make_double4(am[0], am[1], am[2], am[3]));
            st4(rm + n + i, make_double4(am[4], am[5], am[6], am[7]));
            st4(rm + 3 * n + i, make_double4(xv.x, xv.y, xv.z, vol));
        } else {
            st4(rm + i, make_double4(am[0], am[1], am[2], am[3]));
        }
    }
}

// q_a = D rho_l,a sum_b V_b (s_a - s_b) A_a gradW: A_a is per particle, so
// the gather sums sum_b V_b (s_a - s_b) gradW and A_a is applied once
// pack: 1 = write q into the mass-update record (first flux of the outer
// step), 0 = into the flux-rate record (second)
template <int D>
__global__ void __launch_bounds__(256) k_por_flux(PorousArgs A, int pack) {
    const int64_t n = A.n;
    POR_ROWS_BEGIN
    double acc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = 0.0;
    if (act) {
        double xa[3];
        xget<D>(ldg4(A.XV + i), xa);
        const double sa = A.sat[i];
        // (light gather, one record per neighbour: streaming the stored gradient
        // magnitudes as well measured slower, outer step 33.2 -> 40.2 ms at 17 M)
        auto visit = [&](int32_t b) {
            const double4 xvb = ldg4(A.XV + b);
            double xb[3], rel[D], g[D];
            xget<D>(xvb, xb);
#pragma unroll
            for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
            grad_w<D>(rel, A.ks, g);
            const double wgt = A.volc[b] * (sa - A.sat[b]);
#pragma unroll
            for (int c = 0; c < D; ++c) acc[c] += wgt * g[c];
        };
        por_walk(A, i, sub, visit);
    }
    group_sum<kPorLanes>(acc);
    if (act && sub == 0 && !(A.flags[i] & PF_GHOST)) {
        const double cf = A.coeff[i];
        double qv[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) s += A.amap[(int64_t)(r * D + c) * n + i] * acc[c];
            qv[r] = s * cf;
            A.q[(int64_t)r * n + i] = qv[r];
        }
        if (pack) {
            double4 *rm = reinterpret_cast<double4 *>(A.rm);
            if (D == 3) st4(rm + 2 * n + i, make_double4(A.amap[(int64_t)8 * n + i], qv[0], qv[1], qv[2]));
            else st4(rm + n + i, make_double4(qv[0], qv[1], A.volc[i], 0.0));
        } else {
            st4(reinterpret_cast<double4 *>(A.rf) + n + i, make_double4(qv[0], qv[1], qv[2], 0.0));
        }
    }
    POR_ROWS_END
}

// mass update + clamp + contact/evaporation; partial[0][blk] = clamp count
template <int D>
__global__ void __launch_bounds__(256) k_por_mass(PorousArgs A, double dt, int contact_on, double evap_factor) {
    __shared__ double sh[32];
    const int64_t n = A.n;
    double clamped = 0.0;
    POR_ROWS_BEGIN
    double rate[1] = {0.0};
    if (act) {
        double xa[3], ama[D * D], qa[D];
        xget<D>(ldg4(A.XV + i), xa);
#pragma unroll
        for (int k = 0; k < D * D; ++k) ama[k] = A.amap[(int64_t)k * n + i];
#pragma unroll
        for (int k = 0; k < D; ++k) qa[k] = A.q[(int64_t)k * n + i];
        const double4 *rm = reinterpret_cast<const double4 *>(A.rm);
        auto visit = [&](int32_t b) {
            // A_b, q_b, V_b (and X_b in 3D) from the planar record
            double ab[D * D], qb[D], xb[3], vb;
            const double4 p0 = ldg4(rm + b), p1 = ldg4(rm + n + b);
            if (D == 3) {
                const double4 p2 = ldg4(rm + 2 * n + b), p3 = ldg4(rm + 3 * n + b);
                ab[0] = p0.x; ab[1] = p0.y; ab[2] = p0.z; ab[3] = p0.w;
                ab[4] = p1.x; ab[5] = p1.y; ab[6] = p1.z; ab[7] = p1.w;
                ab[8] = p2.x; qb[0] = p2.y; qb[1] = p2.z; qb[2] = p2.w;
                xb[0] = p3.x; xb[1] = p3.y; xb[2] = p3.z; vb = p3.w;
            } else {
                ab[0] = p0.x; ab[1] = p0.y; ab[2] = p0.z; ab[3] = p0.w;
                qb[0] = p1.x; qb[1] = p1.y; vb = p1.z;
                xget<D>(ldg4(A.XV + b), xb);
            }
            double rel[D], g[D];
#pragma unroll
            for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
            grad_w<D>(rel, A.ks, g);
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) s += 0.5 * (ama[r * D + c] + ab[r * D + c]) * g[c];
                acc += (qa[r] + qb[r]) * s;
            }
            rate[0] -= vb * acc;
        };
        por_walk(A, i, sub, visit);
    }
    group_sum<kPorLanes>(rate);
    if (act && sub == 0 && !(A.flags[i] & PF_GHOST)) {
        const double va = A.volc[i];
        double mass = A.mass_l[i] + dt * (va * rate[0]);
        const double cap = A.m.porosity * A.m.rho_l0 * va;
        if (mass < 0.0 || mass > cap) clamped += 1.0;
        mass = fmin(fmax(mass, 0.0), cap);
        if (contact_on) {
            if (A.flags[i] & PF_CONTACT) mass = A.m.porosity * A.m.rho_l0 * va;
        } else if (evap_factor != 1.0) {
            mass = mass * evap_factor;
        }
        A.mass_l[i] = mass;
    }
    POR_ROWS_END
    const double s = block_sum<256>(clamped, sh);
    if (threadIdx.x == 0) A.part[blockIdx.x] = s;
}

// split_velocities (porous.py:266) for particle i; returns v_s, v_l
template <int D>
__device__ __forceinline__ void split_vel(const PorousArgs &A, int64_t i, double j, const double *M,
                                          const double *q, double *vs, double *vl) {
    const double rho_s = A.m.rho_s0 / j;
    const double rho_l = A.mass_l[i] / (volof<D>(A.XV[i]) * j);
    const double rho = rho_s + rho_l;
    const bool dry = rho_l < 1e-12 * A.m.rho_l0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double f = dry ? 0.0 : q[k];
        vs[k] = (M[k] - f) / rho;
        vl[k] = dry ? vs[k] : vs[k] + f / (dry ? 1.0 : rho_l);
    }
    if (!(A.flags[i] & PF_MOVABLE)) {
#pragma unroll
        for (int k = 0; k < D; ++k) { vs[k] = 0.0; vl[k] = 0.0; }
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_por_post(PorousArgs A) {
    using V_t = typename VT<D>::T;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    if (A.flags[i] & PF_GHOST) return;
    const int64_t n = A.n;
    const double sat = A.sat[i];
    A.pres[i] = A.m.C * (sat - A.m.sat0);
    const double mix = A.m.rho_s0 * volof<D>(A.XV[i]) + A.mass_l[i];
    A.mix[i] = mix;
    const bool movable = A.flags[i] & PF_MOVABLE;
    A.inv_mix[i] = movable ? 1.0 / mix : 0.0;
    const double rho_lf = sat * A.m.rho_l0;
    A.rho_lf[i] = rho_lf;
    const double j = A.J[i];
    const double rho = A.m.rho_s0 / j + rho_lf;
    V_t *V = reinterpret_cast<V_t *>(A.V);
    double v0[3], M[D], q[D], vs[D], vl[D];
    vget(V[i], v0);
#pragma unroll
    for (int k = 0; k < D; ++k) {
        q[k] = A.q[(int64_t)k * n + i];
        M[k] = movable ? rho * v0[k] + q[k] : q[k];
        A.M[(int64_t)k * n + i] = M[k];
    }
    split_vel<D>(A, i, j, M, q, vs, vl);
    double v3[3] = {0, 0, 0}, l3[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < D; ++k) {
        v3[k] = vs[k];
        l3[k] = vl[k];
        A.vl[(int64_t)k * n + i] = vl[k];
    }
    st4(reinterpret_cast<double4 *>(A.rf) + i, make_double4(l3[0], l3[1], l3[2], A.volc[i]));
    V_t w;
    vset(w, v3);
    V[i] = w;
}

// -sum_b V_b (vl_a q_a^T + vl_b q_b^T) (A_a gradW) (porous.py:239), with the
// neighbour loop carrying G = sum_b V_b g and sum_b V_b (q_b . g) vl_b,
// g = -A_a gradW: the vl_a q_a^T term is applied once after the loop
template <int D>
__global__ void __launch_bounds__(256, 3) k_por_fluxrate(PorousArgs A) {
    const int64_t n = A.n;
    POR_ROWS_BEGIN
    double acc[2 * D];   // [0, D): sum V_b (q_b.g) vl_b ; [D, 2D): sum V_b g
#pragma unroll
    for (int k = 0; k < 2 * D; ++k) acc[k] = 0.0;
    if (act) {
        double xa[3], am[D * D];
        xget<D>(ldg4(A.XV + i), xa);
#pragma unroll
        for (int k = 0; k < D * D; ++k) am[k] = -A.amap[(int64_t)k * n + i];
        const double4 *rf = reinterpret_cast<const double4 *>(A.rf);
        auto visit = [&](int32_t b) {
            const double4 xvb = ldg4(A.XV + b);
            double xb[3], rel[D], g0[D], g[D];
            xget<D>(xvb, xb);
#pragma unroll
            for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
            grad_w<D>(rel, A.ks, g0);
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) s += am[r * D + c] * g0[c];
                g[r] = s;
            }
            const double4 f0 = ldg4(rf + b), f1 = ldg4(rf + n + b);
            const double vlb[3] = {f0.x, f0.y, f0.z}, qb[3] = {f1.x, f1.y, f1.z};
            const double vb = f0.w;
            double qg = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) qg += qb[c] * g[c];
            const double w = vb * qg;
#pragma unroll
            for (int r = 0; r < D; ++r) {
                acc[r] += w * vlb[r];
                acc[D + r] += vb * g[r];
            }
        };
        por_walk(A, i, sub, visit);
    }
    group_sum<kPorLanes>(acc);
    if (act && sub == 0 && !(A.flags[i] & PF_GHOST)) {
        double qa[D], qG = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) {
            qa[c] = A.q[(int64_t)c * n + i];
            qG += qa[c] * acc[D + c];
        }
#pragma unroll
        for (int r = 0; r < D; ++r) A.frate[(int64_t)r * n + i] = A.vl[(int64_t)r * n + i] * qG + acc[r];
    }
    POR_ROWS_END
}

// ---------------------------------------------------------- inner step

template <int D>
__global__ void __launch_bounds__(256) k_por_kick1(PorousArgs A) {
    using V_t = typename VT<D>::T;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    if (A.flags[i] & PF_GHOST) return;
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const double dt = c->dt;
    const int64_t n = A.n;
    const bool movable = A.flags[i] & PF_MOVABLE;
    const double rho = A.m.rho_s0 / A.J[i] + A.rho_lf[i];
    double v[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double q = A.q[(int64_t)k * n + i];
        double M = A.M[(int64_t)k * n + i] + 0.5 * dt * A.rate[(int64_t)k * n + i];
        if (!movable) M = q;
        A.M[(int64_t)k * n + i] = M;
        v[k] = movable ? (M - q) / rho : 0.0;
        A.x[(int64_t)k * n + i] += dt * v[k];
    }
    V_t w;
    vset(w, v);
    reinterpret_cast<V_t *>(A.V)[i] = w;
}

// J, Almansi mixture stress, nominal stress (porous.py / _accel.py:240),
// divergence record T~ = V0 Pm B with the reference position; element-wise,
// after the gather kernel updated F
template <int D>
__global__ void __launch_bounds__(256) k_por_constit(PorousArgs A) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    if (A.flags[i] & PF_GHOST) return;
    Ctrl *c = A.ctrl;
    if (c->done) return;
    const int64_t n = A.n;
    double F[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) F[k] = A.F[(int64_t)k * n + i];
    const double j = det_d<D>(F);
    A.J[i] = j;
    double Tm[D * D];
    if (!(j > 0.0)) {
        atomicMin(&c->err_inv, (unsigned long long)A.perm[i]);
#pragma unroll
        for (int k = 0; k < D * D; ++k) Tm[k] = 0.0;
    } else {
        double fi[D * D], e[D * D], sg[D * D], pm[D * D], Bm[D * D];
        inv_d<D>(F, j, fi);
        double tre = 0.0;
#pragma unroll
        for (int r = 0; r < D; ++r) {
#pragma unroll
            for (int cc = 0; cc < D; ++cc) {
                double s = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) s += fi[k * D + r] * fi[k * D + cc];
                e[r * D + cc] = -0.5 * s;
            }
            e[r * D + r] += 0.5;
            tre += e[r * D + r];
        }
        const double dia = A.m.lam * tre - A.pres[i];
#pragma unroll
        for (int k = 0; k < D * D; ++k) sg[k] = 2.0 * A.m.mu * e[k];
#pragma unroll
        for (int r = 0; r < D; ++r) sg[r * D + r] += dia;
        double tmp[D * D];
        mmt<D>(sg, fi, tmp);  // sigma F^-T
#pragma unroll
        for (int k = 0; k < D * D; ++k) pm[k] = j * tmp[k];
#pragma unroll
        for (int k = 0; k < D * D; ++k) Bm[k] = A.B[(int64_t)k * n + i];
        mm<D>(pm, Bm, Tm);
    }
    const double4 xv = ldg4(A.XV + i);
    const double vol = volof<D>(xv);
#pragma unroll
    for (int k = 0; k < D * D; ++k) Tm[k] *= vol;
    dstore_raw<D>(A.T, n, i, Tm, xv);
}

// sum_b V_b gradW_ab per particle (static; once at setup), CSR row order
template <int D>
__global__ void __launch_bounds__(256) k_por_gsum(PorousArgs A, double *G) {
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
__global__ void __launch_bounds__(256, 3) k_por_stress(PorousArgs A) {
    using V_t = typename VT<D>::T;
    Ctrl *c = A.ctrl;
    if (c->done) return;
    const double dt = c->dt;
    const int64_t n = A.n;
    const V_t *V = reinterpret_cast<const V_t *>(A.V);
    POR_ROWS_BEGIN
    double acc[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) acc[k] = 0.0;
    if (act) {
        double xa[3], va[3];
        xget<D>(ldg4(A.XV + i), xa);
        vget(vldg(V + i), va);
        auto visit = [&](int32_t b, double mag) {
            const double4 xvb = ldg4(A.XV + b);
            double xb[3], vb[3], rel[D], g[D];
            xget<D>(xvb, xb);
            vget(vldg(V + b), vb);
#pragma unroll
            for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
            if (MTSPH_POR_STRESS_MAG) grad_w_mag<D>(rel, A.ks, mag, g);
            else grad_w<D>(rel, A.ks, g);
            const double volb = volof<D>(xvb);
#pragma unroll
            for (int r = 0; r < D; ++r) {
                const double dv = volb * (vb[r] - va[r]);
#pragma unroll
                for (int cc = 0; cc < D; ++cc) acc[r * D + cc] += dv * g[cc];
            }
        };
        if (MTSPH_POR_STRESS_MAG) por_walk_mag<false>(A, i, sub, visit);
        else por_walk<false>(A, i, sub, [&](int32_t b) { visit(b, 0.0); });
    }
    group_sum<kPorLanes>(acc);
    if (act && sub == 0 && !(A.flags[i] & PF_GHOST)) {  // F += dt (acc B)
        double Bm[D * D], L[D * D];
#pragma unroll
        for (int k = 0; k < D * D; ++k) Bm[k] = A.B[(int64_t)k * n + i];
        mm<D>(acc, Bm, L);
#pragma unroll
        for (int k = 0; k < D * D; ++k) A.F[(int64_t)k * n + i] += dt * L[k];
    }
    POR_ROWS_END
}


template <int D>
__global__ void __launch_bounds__(256, 3) k_por_accel(PorousArgs A) {
    using V_t = typename VT<D>::T;
    __shared__ double sh[32];
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const int64_t n = A.n;
    const double dt = c->dt;
    double ek = 0.0, a2m = 0.0;
    POR_ROWS_BEGIN
    // sum_b V_b (T_a + T_b) gradW = sum_b T~_b gradW + T_a G_a, with the
    // divergence record T~_b = V_b T_b (three 256-bit loads per neighbour,
    // X included) and G_a = sum_b V_b gradW static
    double acc[D];
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = 0.0;
    if (act) {
        double xa[3];
        xget<D>(ldg4(A.XV + i), xa);
        auto visit = [&](int32_t b) {
            double xb[3], Tb[D * D], rel[D], g[D];
            dload<D>(A.T, n, A.XV, b, Tb, xb);
#pragma unroll
            for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
            grad_w<D>(rel, A.ks, g);
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
                for (int cc = 0; cc < D; ++cc) acc[r] = fma(Tb[r * D + cc], g[cc], acc[r]);
        };
        por_walk(A, i, sub, visit);
    }
    group_sum<kPorLanes>(acc);
    if (act && sub == 0 && !(A.flags[i] & PF_GHOST)) {
        double Ta[D * D], xd[3];
        dload<D>(A.T, n, A.XV, i, Ta, xd);
        const double vola = volof<D>(ldg4(A.XV + i));
        const bool movable = A.flags[i] & PF_MOVABLE;
        const double rho = A.m.rho_s0 / A.J[i] + A.rho_lf[i];
        const double rmix = A.mix[i] / volof<D>(ldg4(A.XV + i));
        double v[3] = {0, 0, 0}, v2 = 0.0, aa = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            double ta = 0.0;
#pragma unroll
            for (int cc = 0; cc < D; ++cc) ta += Ta[k * D + cc] * A.G[(int64_t)cc * n + i];
            const double rt = acc[k] + ta / vola + A.frate[(int64_t)k * n + i];
            A.rate[(int64_t)k * n + i] = rt;
            const double q = A.q[(int64_t)k * n + i];
            double M = A.M[(int64_t)k * n + i] + 0.5 * dt * rt;
            if (!movable) M = q;
            A.M[(int64_t)k * n + i] = M;
            v[k] = movable ? (M - q) / rho : 0.0;
            v2 += v[k] * v[k];
            aa += rt * rt;
        }
        V_t w2;
        vset(w2, v);
        reinterpret_cast<V_t *>(A.V)[i] = w2;
        if (movable) {
            ek += A.mix[i] * v2;
            a2m = fmax(a2m, aa / (rmix * rmix));
        }
    }
    POR_ROWS_END
    const double se = block_sum<256>(ek, sh);
    const double sa = block_max<256>(a2m, sh);
    if (threadIdx.x == 0) {
        A.part[blockIdx.x] = se;
        A.part[A.nblk + blockIdx.x] = sa;
    }
}

// momentum rebuild after damping + |v|^2 max; with_accel = 1 is the
// pre-loop reduction (no rebuild; |a|^2 of the free particles)
template <int D>
__global__ void __launch_bounds__(256) k_por_post_step(PorousArgs A, int pre_loop) {
    using V_t = typename VT<D>::T;
    __shared__ double sh[32];
    if (!pre_loop && A.ctrl->done) return;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n = A.n;
    double v2 = 0.0, a2 = 0.0;
    if (i < n && !(A.flags[i] & PF_GHOST)) {
        double v[3];
        vget(reinterpret_cast<const V_t *>(A.V)[i], v);
        const bool movable = A.flags[i] & PF_MOVABLE;
        if (!pre_loop) {
            const double rho = A.m.rho_s0 / A.J[i] + A.rho_lf[i];
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const double q = A.q[(int64_t)k * n + i];
                A.M[(int64_t)k * n + i] = movable ? rho * v[k] + q : q;
            }
        } else if (movable) {
            const double rmix = A.mix[i] / volof<D>(A.XV[i]);
            double aa = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const double r = A.rate[(int64_t)k * n + i];
                aa += r * r;
            }
            a2 = aa / (rmix * rmix);
        }
#pragma unroll
        for (int k = 0; k < D; ++k) v2 += v[k] * v[k];
    }
    const double mv = block_max<256>(v2, sh);
    const double ma = block_max<256>(a2, sh);
    if (threadIdx.x == 0) {
        A.part[2 * A.nblk + blockIdx.x] = mv;
        if (pre_loop) A.part[A.nblk + blockIdx.x] = ma;
    }
}

// measure(): split_velocities refresh (vel_solid, vel_fluid) from M and q
template <int D>
__global__ void __launch_bounds__(256) k_por_refresh(PorousArgs A) {
    using V_t = typename VT<D>::T;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const int64_t n = A.n;
    double F[D * D], M[D], q[D], vs[D], vl[D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) F[k] = A.F[(int64_t)k * n + i];
    const double j = det_d<D>(F);
#pragma unroll
    for (int k = 0; k < D; ++k) {
        M[k] = A.M[(int64_t)k * n + i];
        q[k] = A.q[(int64_t)k * n + i];
    }
    split_vel<D>(A, i, j, M, q, vs, vl);
    double v3[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < D; ++k) {
        v3[k] = vs[k];
        A.vl[(int64_t)k * n + i] = vl[k];
    }
    V_t w;
    vset(w, v3);
    reinterpret_cast<V_t *>(A.V)[i] = w;
}

}  // namespace mtsph

namespace mtsph {

// multi-rank field exchange: 0 vel (d), 1 T~ (d*d; the receiver keeps its
// own copy of X), 2 (s, V) (2), 3 mass-update record (16 / 8), 4 flux-rate
// record (8), 5 1/m_mix (1)
inline int por_field_width(int which, int d) {
    switch (which) {
    case 0: return d;
    case 1: return d * d;
    case 2: return 2;
    case 3: return d == 3 ? 16 : 8;
    case 4: return 8;
    default: return 1;
    }
}

template <int D>
__global__ void k_por_pack(PorousArgs A, int64_t m, const int64_t *__restrict__ ids, int which, int w,
                           double *buf, int unpack) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int64_t i = ids[k], n = A.n;
    double *e = buf + k * w;
    using V_t = typename VT<D>::T;
    if (which == 0) {
        V_t *V = reinterpret_cast<V_t *>(A.V);
        if (unpack) {
            double v[3] = {0, 0, 0};
            for (int c = 0; c < D; ++c) v[c] = e[c];
            V_t o;
            vset(o, v);
            V[i] = o;
        } else {
            double v[3];
            vget(V[i], v);
            for (int c = 0; c < D; ++c) e[c] = v[c];
        }
    } else if (which == 1) {
        double t[D * D], x[3];
        if (unpack) {
            for (int c = 0; c < D * D; ++c) t[c] = e[c];
            dstore_raw<D>(A.T, n, i, t, A.XV[i]);
        } else {
            dload<D>(A.T, n, A.XV, i, t, x);
            for (int c = 0; c < D * D; ++c) e[c] = t[c];
        }
    } else if (which == 2) {
        if (unpack) { A.sat[i] = e[0]; A.volc[i] = e[1]; }
        else { e[0] = A.sat[i]; e[1] = A.volc[i]; }
    } else if (which == 3 || which == 4) {
        const int planes = w / 4;
        double4 *r = reinterpret_cast<double4 *>(which == 3 ? A.rm : A.rf);
        for (int p = 0; p < planes; ++p) {
            if (unpack) r[p * n + i] = make_double4(e[4 * p], e[4 * p + 1], e[4 * p + 2], e[4 * p + 3]);
            else {
                const double4 q = r[p * n + i];
                e[4 * p] = q.x; e[4 * p + 1] = q.y; e[4 * p + 2] = q.z; e[4 * p + 3] = q.w;
            }
        }
    } else {
        if (unpack) A.inv_mix[i] = e[0];
        else e[0] = A.inv_mix[i];
    }
}

}  // namespace mtsph
