// damping.cuh -- pairwise implicit viscous damping sweeps (paper Eq. 24-25,
// §4.3 pairwise splitting; reference _accel.py:97-206).
//
// Every group of pairs is solved with backward Euler in closed form (one
// pair) or by a small Gaussian elimination (mirror-image pairs that share
// particles, solved simultaneously as in the reference).  The sweep visits
// all groups forward then in reverse, half the step each.
//
//  * serial  : the reference's exact group sequence, level-scheduled; the
//              groups of one level touch disjoint particles, so running a
//              level in parallel performs exactly the serial operations.
//              One CTA walks all levels (__syncthreads between levels).
//  * coloured: groups bucketed into midpoint-cell tasks of 3^d colours;
//              one kernel per colour and direction, one thread per task,
//              groups of a task in the reference's within-task order.
//
// The damping coefficient 2 V_i V_j (-e.gradW)/r of each pair
// (neighbors.py:137-144) is recomputed from the reference positions in the
// kernel instead of being streamed from HBM.
#pragma once

#include "common.cuh"
#include "nbh.cuh"

namespace mtsph {

struct Ctrl {
    double dt, eta, cfl, criterion, dt_outer;
    double ek, vmax2, amax2, min_dt, last_dt;
    double ramp_disp, h, sound;
    double vol_movable;   // porous energy density normaliser
    long long n_inner, min_inner, max_inner, ramp_left;
    int done, cap_hit, mode;
    int remote_err;       // multi-rank: another rank reported an error (k_ctrl_ranks)
    unsigned long long err_inv, err_rm;  // min original id per error class
};

template <int D> struct VT;
template <> struct VT<2> { using T = double2; };
template <> struct VT<3> { using T = double4; };

__device__ __forceinline__ void vget(const double2 &v, double *o) { o[0] = v.x; o[1] = v.y; }
__device__ __forceinline__ void vget(const double4 &v, double *o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; }
// read-only velocity record (kernels that do not write V)
__device__ __forceinline__ double2 vldg(const double2 *p) { return __ldg(p); }
__device__ __forceinline__ double4 vldg(const double4 *p) { return ldg4(p); }
__device__ __forceinline__ double2 vldcg(const double2 *p) { return __ldcg(p); }
__device__ __forceinline__ double4 vldcg(const double4 *p) { return ldcg4(p); }
__device__ __forceinline__ void vst(double2 *p, const double2 &v) { *p = v; }
__device__ __forceinline__ void vst(double4 *p, const double4 &v) { st4(p, v); }
__device__ __forceinline__ void vset(double2 &v, const double *o) { v.x = o[0]; v.y = o[1]; }
__device__ __forceinline__ void vset(double4 &v, const double *o) { v.x = o[0]; v.y = o[1]; v.z = o[2]; v.w = 0.0; }

// fp32 variant (solid32.cuh): the same records in single precision
template <int D, class R> struct VTR { using T = typename VT<D>::T; };
template <> struct VTR<2, float> { using T = float2; };
template <> struct VTR<3, float> { using T = float4; };
__device__ __forceinline__ void vget(const float2 &v, float *o) { o[0] = v.x; o[1] = v.y; }
__device__ __forceinline__ void vget(const float4 &v, float *o) { o[0] = v.x; o[1] = v.y; o[2] = v.z; }
__device__ __forceinline__ float2 vldg(const float2 *p) { return __ldg(p); }
__device__ __forceinline__ float4 vldg(const float4 *p) { return __ldg(p); }
__device__ __forceinline__ float2 vldcg(const float2 *p) { return __ldcg(p); }
__device__ __forceinline__ float4 vldcg(const float4 *p) { return __ldcg(p); }
__device__ __forceinline__ void vst(float2 *p, const float2 &v) { *p = v; }
__device__ __forceinline__ void vst(float4 *p, const float4 &v) { *p = v; }
__device__ __forceinline__ void vset(float2 &v, const float *o) { v.x = o[0]; v.y = o[1]; }
__device__ __forceinline__ void vset(float4 &v, const float *o) { v.x = o[0]; v.y = o[1]; v.z = o[2]; v.w = 0.f; }

template <int D> __device__ __forceinline__ void xget(const double4 &xv, double *x) {
    x[0] = xv.x; x[1] = xv.y;
    if (D == 3) x[2] = xv.z;
}
template <int D> __device__ __forceinline__ double volof(const double4 &xv) { return D == 3 ? xv.w : xv.z; }

// neighbors.py:137-144: 2 V_i V_j (-(e . grad W_ij)) / |r_ij|, r = X_j - X_i
template <int D>
__device__ __forceinline__ double pair_damp(const double4 &xi, const double4 &xj, const KSpec &ks) {
    double a[3], b[3], rel[D], g[D];
    xget<D>(xi, a);
    xget<D>(xj, b);
    double r2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { rel[k] = b[k] - a[k]; r2 += rel[k] * rel[k]; }
    const double r = sqrt(r2);
    grad_w<D>(rel, ks, g);
    double radial = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) radial -= (rel[k] / r) * g[k];
    return 2.0 * volof<D>(xi) * volof<D>(xj) * radial / r;
}

struct SweepArgs {
    const int32_t *pi, *pj;
    const int64_t *gptr, *gscr;
    double *scratch;
    const double4 *XV;
    const double *inv_m;
    void *V;
    KSpec ks;
};

// CG: read the velocities through L2 (the multi-CTA serial kernel, where
// other SMs wrote them at earlier levels)
template <int D, bool CG = false>
__device__ __forceinline__ void visit_group(const SweepArgs &A, int64_t g, double half) {
    using V_t = typename VT<D>::T;
    V_t *V = reinterpret_cast<V_t *>(A.V);
    auto vload = [&](int64_t i) { return CG ? vldcg(V + i) : V[i]; };
    const int64_t lo = A.gptr[g], hi = A.gptr[g + 1];
    if (hi - lo == 1) {
        const int32_t i = A.pi[lo], j = A.pj[lo];
        const double c = half * pair_damp<D>(A.XV[i], A.XV[j], A.ks);
        const double ca = c * A.inv_m[i], cb = c * A.inv_m[j];
        const double den = 1.0 + ca + cb;
        V_t vi = vload(i), vj = vload(j);
        double a[3], b[3];
        vget(vi, a);
        vget(vj, b);
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const double u = (a[m] - b[m]) / den;
            a[m] -= ca * u;
            b[m] += cb * u;
        }
        vset(vi, a);
        vset(vj, b);
        V[i] = vi;
        V[j] = vj;
        return;
    }
    // simultaneous solve (_accel.py:107), scratch: A[nb*nb] rhs[nb*3] loc[nb]
    double *S = A.scratch + A.gscr[g];
    const int nbmax = (int)(2 * (hi - lo));
    double *Am = S;
    double *rhs = S + nbmax * nbmax;
    long long *loc = reinterpret_cast<long long *>(rhs + 3 * nbmax);
    int nb = 0;
    for (int64_t k = lo; k < hi; ++k) {
        const int32_t e[2] = {A.pi[k], A.pj[k]};
        for (int s = 0; s < 2; ++s) {
            bool found = false;
            for (int t = 0; t < nb; ++t) if (loc[t] == e[s]) { found = true; break; }
            if (!found) loc[nb++] = e[s];
        }
    }
    for (int r = 0; r < nb; ++r) {
        for (int c = 0; c < nb; ++c) Am[r * nb + c] = (r == c) ? 1.0 : 0.0;
        double v[3];
        vget(vload(loc[r]), v);
        for (int m = 0; m < D; ++m) rhs[r * 3 + m] = v[m];
    }
    for (int64_t k = lo; k < hi; ++k) {
        const int32_t i = A.pi[k], j = A.pj[k];
        const double c = half * pair_damp<D>(A.XV[i], A.XV[j], A.ks);
        int ia = 0, ib = 0;
        for (int t = 0; t < nb; ++t) {
            if (loc[t] == i) ia = t;
            if (loc[t] == j) ib = t;
        }
        const double ca = c * A.inv_m[i], cb = c * A.inv_m[j];
        Am[ia * nb + ia] += ca;
        Am[ia * nb + ib] -= ca;
        Am[ib * nb + ib] += cb;
        Am[ib * nb + ia] -= cb;
    }
    for (int col = 0; col < nb - 1; ++col) {
        const double piv = Am[col * nb + col];
        for (int r = col + 1; r < nb; ++r) {
            const double f = Am[r * nb + col] / piv;
            if (f != 0.0) {
                for (int c = col; c < nb; ++c) Am[r * nb + c] -= f * Am[col * nb + c];
                for (int m = 0; m < D; ++m) rhs[r * 3 + m] -= f * rhs[col * 3 + m];
            }
        }
    }
    for (int r = nb - 1; r >= 0; --r)
        for (int m = 0; m < D; ++m) {
            double s = rhs[r * 3 + m];
            for (int c = r + 1; c < nb; ++c) s -= Am[r * nb + c] * rhs[c * 3 + m];
            rhs[r * 3 + m] = s / Am[r * nb + r];
        }
    for (int t = 0; t < nb; ++t) {
        double v[3] = {rhs[t * 3], rhs[t * 3 + 1], rhs[t * 3 + 2]};
        V_t w;
        vset(w, v);
        V[loc[t]] = w;
    }
}

// exact serial order: one CTA walks the levels forward, then backward
template <int D>
__global__ void __launch_bounds__(1024) k_sweep_serial(SweepArgs A, const int64_t *__restrict__ level_ptr,
                                                       int64_t nlevels, const int64_t *__restrict__ level_groups,
                                                       const Ctrl *ctrl) {
    if (ctrl->done) return;
    const double half = 0.5 * ctrl->dt * ctrl->eta;
    for (int64_t L = 0; L < nlevels; ++L) {
        for (int64_t k = level_ptr[L] + threadIdx.x; k < level_ptr[L + 1]; k += blockDim.x)
            visit_group<D>(A, level_groups[k], half);
        __syncthreads();
    }
    for (int64_t L = nlevels - 1; L >= 0; --L) {
        for (int64_t k = level_ptr[L] + threadIdx.x; k < level_ptr[L + 1]; k += blockDim.x)
            visit_group<D>(A, level_groups[k], half);
        __syncthreads();
    }
}

// ---- exact serial order, small problems: velocities and the level table
// in shared memory.  The global kernel above pays a chain of dependent L2
// loads per level (level table -> group -> pair -> positions -> velocity)
// before its barrier; here the velocities live in shared memory and each
// thread's single-pair entries of the next levels (i, j and the static
// pair_damp, precomputed in level order by k_serial_entries) are loaded
// ahead through a register ring.  Groups of 2..kGroupMax pairs (the
// reference's simultaneous solves of mirror pairs) are solved from their
// precomputed entries in local arrays; larger ones take the global path's
// solver on the shared copy.  Same operations in the same order:
// bit-identical to k_sweep_serial (tests/test_gpu_sweeps.py
// test_serial_sweep_shared_memory_kernel_is_bit_identical*).  Most levels
// hold one small group, whose dependent solve (~3 us) is now the critical
// path between two barriers.

// entry k (level order): a single pair -> (i | j << 32, pair_damp); a group
// of 2..kGroupMax pairs -> (-2 - (side offset << 8 | count), 0) with its
// pairs' (i | j << 32, pair_damp) at side[offset ...]; a larger group ->
// (-2 - (g << 8), 0) (count 0: the global solver)
constexpr int kGroupMax = 8;

__device__ __forceinline__ double2 pair_entry(int32_t i, int32_t j, double pd) {
    const unsigned long long ij = (unsigned long long)(uint32_t)i | ((unsigned long long)(uint32_t)j << 32);
    return make_double2(__longlong_as_double((long long)ij), pd);
}

template <int D>
__global__ void k_serial_entries(SweepArgs A, const int64_t *__restrict__ level_groups, int64_t ng,
                                 const int64_t *__restrict__ side_off, double2 *out, double2 *side) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= ng) return;
    const int64_t g = level_groups[k];
    const int64_t lo = A.gptr[g], hi = A.gptr[g + 1];
    if (hi - lo == 1) {
        const int32_t i = A.pi[lo], j = A.pj[lo];
        out[k] = pair_entry(i, j, pair_damp<D>(A.XV[i], A.XV[j], A.ks));
    } else if (hi - lo <= kGroupMax) {
        const int64_t o = side_off[k];
        for (int64_t q = lo; q < hi; ++q) {
            const int32_t i = A.pi[q], j = A.pj[q];
            side[o + (q - lo)] = pair_entry(i, j, pair_damp<D>(A.XV[i], A.XV[j], A.ks));
        }
        out[k] = make_double2(__longlong_as_double(-2 - ((o << 8) | (hi - lo))), 0.0);
    } else {
        out[k] = make_double2(__longlong_as_double(-2 - (g << 8)), 0.0);
    }
}

// the simultaneous solve of a small group from its precomputed pair
// entries, local arrays instead of the global scratch (same arithmetic as
// visit_group)
template <int D, class Acc>
__device__ void group_solve_entries_acc(const double2 *__restrict__ pe, int cnt, const double *__restrict__ inv_m,
                                        double half, const Acc &V) {
    constexpr int NB = 2 * kGroupMax;
    double2 e[kGroupMax];
    for (int q = 0; q < cnt; ++q) e[q] = __ldg(pe + q);
    int ii[kGroupMax], jj[kGroupMax];
    double imi[kGroupMax], imj[kGroupMax];
    for (int q = 0; q < cnt; ++q) {
        const unsigned long long key = (unsigned long long)__double_as_longlong(e[q].x);
        ii[q] = (int)(uint32_t)key;
        jj[q] = (int)(uint32_t)(key >> 32);
    }
    for (int q = 0; q < cnt; ++q) {
        imi[q] = __ldg(inv_m + ii[q]);
        imj[q] = __ldg(inv_m + jj[q]);
    }
    int loc[NB];
    int nb = 0;
    for (int q = 0; q < cnt; ++q) {
        const int ep[2] = {ii[q], jj[q]};
        for (int s = 0; s < 2; ++s) {
            bool found = false;
            for (int t = 0; t < nb; ++t) if (loc[t] == ep[s]) { found = true; break; }
            if (!found) loc[nb++] = ep[s];
        }
    }
    double Am[NB * NB], rhs[NB * 3];
    for (int r = 0; r < nb; ++r) {
        for (int c = 0; c < nb; ++c) Am[r * nb + c] = (r == c) ? 1.0 : 0.0;
        for (int m = 0; m < D; ++m) rhs[r * 3 + m] = V.get(loc[r], m);
    }
    for (int q = 0; q < cnt; ++q) {
        const double c = half * e[q].y;
        int ia = 0, ib = 0;
        for (int t = 0; t < nb; ++t) {
            if (loc[t] == ii[q]) ia = t;
            if (loc[t] == jj[q]) ib = t;
        }
        const double ca = c * imi[q], cb = c * imj[q];
        Am[ia * nb + ia] += ca;
        Am[ia * nb + ib] -= ca;
        Am[ib * nb + ib] += cb;
        Am[ib * nb + ia] -= cb;
    }
    for (int col = 0; col < nb - 1; ++col) {
        const double piv = Am[col * nb + col];
        for (int r = col + 1; r < nb; ++r) {
            const double f = Am[r * nb + col] / piv;
            if (f != 0.0) {
                for (int c = col; c < nb; ++c) Am[r * nb + c] -= f * Am[col * nb + c];
                for (int m = 0; m < D; ++m) rhs[r * 3 + m] -= f * rhs[col * 3 + m];
            }
        }
    }
    for (int r = nb - 1; r >= 0; --r)
        for (int m = 0; m < D; ++m) {
            double s = rhs[r * 3 + m];
            for (int c = r + 1; c < nb; ++c) s -= Am[r * nb + c] * rhs[c * 3 + m];
            rhs[r * 3 + m] = s / Am[r * nb + r];
        }
    for (int t = 0; t < nb; ++t)
        for (int m = 0; m < D; ++m) V.set(loc[t], m, rhs[t * 3 + m]);
}

// velocity accessors of the entry solvers: the shared copy (planar [D][n])
// and the global records read through L2 (multi-CTA kernel: other SMs
// wrote them at earlier levels, so L1 may hold stale lines)
struct PlanarV {
    double *sv;
    int n;
    __device__ __forceinline__ double get(int i, int m) const { return sv[m * n + i]; }
    __device__ __forceinline__ void set(int i, int m, double x) const { sv[m * n + i] = x; }
};

template <int D>
__device__ void group_solve_entries(const double2 *__restrict__ pe, int cnt, const double *__restrict__ inv_m,
                                    double half, double *sv, int n) {
    group_solve_entries_acc<D>(pe, cnt, inv_m, half, PlanarV{sv, n});
}

// velocity accessor of the shared copy: planar [D][n]
struct SmemV {
    double *sv;
    int n;
    __device__ void get(int64_t i, double *a, int D) const { for (int m = 0; m < D; ++m) a[m] = sv[m * n + i]; }
    __device__ void set(int64_t i, const double *a, int D) const { for (int m = 0; m < D; ++m) sv[m * n + i] = a[m]; }
};

// visit_group's simultaneous solve on the shared copy (same arithmetic)
template <int D>
__device__ void group_solve_smem(const SweepArgs &A, int64_t g, double half, const SmemV &V) {
    const int64_t lo = A.gptr[g], hi = A.gptr[g + 1];
    double *S = A.scratch + A.gscr[g];
    const int nbmax = (int)(2 * (hi - lo));
    double *Am = S;
    double *rhs = S + nbmax * nbmax;
    long long *loc = reinterpret_cast<long long *>(rhs + 3 * nbmax);
    int nb = 0;
    for (int64_t k = lo; k < hi; ++k) {
        const int32_t e[2] = {A.pi[k], A.pj[k]};
        for (int s = 0; s < 2; ++s) {
            bool found = false;
            for (int t = 0; t < nb; ++t) if (loc[t] == e[s]) { found = true; break; }
            if (!found) loc[nb++] = e[s];
        }
    }
    for (int r = 0; r < nb; ++r) {
        for (int c = 0; c < nb; ++c) Am[r * nb + c] = (r == c) ? 1.0 : 0.0;
        double v[3];
        V.get(loc[r], v, D);
        for (int m = 0; m < D; ++m) rhs[r * 3 + m] = v[m];
    }
    for (int64_t k = lo; k < hi; ++k) {
        const int32_t i = A.pi[k], j = A.pj[k];
        const double c = half * pair_damp<D>(A.XV[i], A.XV[j], A.ks);
        int ia = 0, ib = 0;
        for (int t = 0; t < nb; ++t) {
            if (loc[t] == i) ia = t;
            if (loc[t] == j) ib = t;
        }
        const double ca = c * A.inv_m[i], cb = c * A.inv_m[j];
        Am[ia * nb + ia] += ca;
        Am[ia * nb + ib] -= ca;
        Am[ib * nb + ib] += cb;
        Am[ib * nb + ia] -= cb;
    }
    for (int col = 0; col < nb - 1; ++col) {
        const double piv = Am[col * nb + col];
        for (int r = col + 1; r < nb; ++r) {
            const double f = Am[r * nb + col] / piv;
            if (f != 0.0) {
                for (int c = col; c < nb; ++c) Am[r * nb + c] -= f * Am[col * nb + c];
                for (int m = 0; m < D; ++m) rhs[r * 3 + m] -= f * rhs[col * 3 + m];
            }
        }
    }
    for (int r = nb - 1; r >= 0; --r)
        for (int m = 0; m < D; ++m) {
            double s = rhs[r * 3 + m];
            for (int c = r + 1; c < nb; ++c) s -= Am[r * nb + c] * rhs[c * 3 + m];
            rhs[r * 3 + m] = s / Am[r * nb + r];
        }
    for (int t = 0; t < nb; ++t) {
        const double v[3] = {rhs[t * 3], rhs[t * 3 + 1], rhs[t * 3 + 2]};
        V.set(loc[t], v, D);
    }
}

constexpr int kSerialThreads = 1024;
constexpr size_t kSerialSmemMax = 200 * 1024;

inline size_t serial_smem_bytes(int64_t n, int d, int64_t nlevels) {
    return (size_t)n * d * sizeof(double) + (size_t)(nlevels + 1) * sizeof(int64_t);
}

template <int D>
__global__ void __launch_bounds__(kSerialThreads, 1)
    k_sweep_serial_smem(SweepArgs A, const double2 *__restrict__ ent, const double2 *__restrict__ side,
                        const int64_t *__restrict__ level_ptr, int64_t nlevels, int n, const Ctrl *ctrl) {
    if (ctrl->done) return;
    extern __shared__ double smem_serial[];
    using V_t = typename VT<D>::T;
    V_t *Vg = reinterpret_cast<V_t *>(A.V);
    const SmemV V{smem_serial, n};
    int64_t *lp = reinterpret_cast<int64_t *>(smem_serial + (size_t)D * n);
    const double half = 0.5 * ctrl->dt * ctrl->eta;
    const int t = threadIdx.x;
    for (int i = t; i < n; i += kSerialThreads) {
        double a[3];
        vget(Vg[i], a);
        V.set(i, a, D);
    }
    for (int64_t L = t; L <= nlevels; L += kSerialThreads) lp[L] = level_ptr[L];
    __syncthreads();
    const double2 none = make_double2(__longlong_as_double(-1ll), 0.0);   // no entry
    auto apply = [&](const double2 &e, double imi, double imj) {
        const long long key = __double_as_longlong(e.x);
        if (key == -1) return;
        if (key < 0) {
            const long long code = -2 - key;
            const int cnt = (int)(code & 0xff);
            if (cnt) group_solve_entries<D>(side + (code >> 8), cnt, A.inv_m, half, smem_serial, n);
            else group_solve_smem<D>(A, code >> 8, half, V);
            return;
        }
        const int i = (int)(uint32_t)key, j = (int)(uint32_t)((unsigned long long)key >> 32);
        const double c = half * e.y;
        const double ca = c * imi, cb = c * imj;
        const double den = 1.0 + ca + cb;
        double a[3], b[3];
        V.get(i, a, D);
        V.get(j, b, D);
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const double u = (a[m] - b[m]) / den;
            a[m] -= ca * u;
            b[m] += cb * u;
        }
        V.set(i, a, D);
        V.set(j, b, D);
    };
    auto inv_of = [&](const double2 &e, double &imi, double &imj) {
        const long long key = __double_as_longlong(e.x);
        imi = imj = 0.0;
        if (key >= 0) {
            imi = __ldg(A.inv_m + (uint32_t)key);
            imj = __ldg(A.inv_m + (uint32_t)((unsigned long long)key >> 32));
        }
    };
    for (int pass = 0; pass < 2; ++pass) {
        // step s visits level s (forward) or nlevels - 1 - s (reverse)
        auto level = [&](int64_t s) { return pass == 0 ? s : nlevels - 1 - s; };
        auto fetch = [&](int64_t s) {
            if (s >= nlevels) return none;
            const int64_t L = level(s), k = lp[L] + t;
            return k < lp[L + 1] ? __ldg(ent + k) : none;
        };
        // ring: entries of steps s..s+3, inverse masses of steps s and s+1
        double2 e0 = fetch(0), e1 = fetch(1), e2 = fetch(2), e3 = fetch(3);
        double i0a, i0b, i1a, i1b;
        inv_of(e0, i0a, i0b);
        inv_of(e1, i1a, i1b);
        for (int64_t s = 0; s < nlevels; ++s) {
            apply(e0, i0a, i0b);
            const int64_t L = level(s);
            for (int64_t k = lp[L] + t + kSerialThreads; k < lp[L + 1]; k += kSerialThreads) {
                const double2 e = __ldg(ent + k);
                double a, b;
                inv_of(e, a, b);
                apply(e, a, b);
            }
            e0 = e1; i0a = i1a; i0b = i1b;
            e1 = e2;
            inv_of(e1, i1a, i1b);
            e2 = e3;
            e3 = fetch(s + 4);
            __syncthreads();
        }
    }
    for (int i = t; i < n; i += kSerialThreads) {
        double a[3];
        V.get(i, a, D);
        V_t w = Vg[i];
        vset(w, a);
        Vg[i] = w;
    }
}

// ---- exact serial order, large problems: every level is spread over the
// whole grid (one persistent launch, all CTAs co-resident) and a grid-wide
// barrier separates consecutive levels.  The levels of the reference order
// grow with the bar length (~30 per lattice column in 3D), the groups of one
// level with the cross-section, so a level of a 10 M-particle bar holds ~1e4
// groups: enough for every SM, where the one-CTA kernels above run them 1024
// at a time.  Entries and arithmetic are those of k_sweep_serial_smem (single
// pairs from the precomputed (i, j, pair_damp) entries, small groups from
// local arrays, larger groups through visit_group); velocities are read
// through L2 (ld.global.cg) because other SMs wrote them at earlier levels.
// Bit-identical to k_sweep_serial (tests/test_gpu_sweeps.py).

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Grid barrier on a monotonic arrival counter, zeroed before the launch:
// barrier k completes when the counter reaches (k + 1) * gridDim.x.  One
// release-add per CTA and a spin on the same word (no separate reset and
// release round trips).
#ifndef MTSPH_GRID_BARRIER_FENCE
#define MTSPH_GRID_BARRIER_FENCE 0
#endif
__device__ __forceinline__ void grid_barrier(unsigned long long *cnt, unsigned long long &target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
#if MTSPH_GRID_BARRIER_FENCE
        __threadfence();
#endif
        // release at gpu scope is cumulative: it orders the CTA's writes that
        // the barrier above made happen-before this thread
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
        while (ld_acquire_u64(cnt) < target) {
        }
    }
    __syncthreads();
}

// global velocity records as an entry-solver accessor
template <int D> struct GlobalV {
    using V_t = typename VT<D>::T;
    V_t *V;
    __device__ __forceinline__ double get(int i, int m) const {
        double a[3];
        vget(vldcg(V + i), a);
        return a[m];
    }
    __device__ __forceinline__ void set(int i, int m, double x) const {
        double *r = reinterpret_cast<double *>(V + i);
        __stcg(r + m, x);
    }
};

constexpr int kSerialGridThreads = 256;

template <int D>
__device__ __forceinline__ void serial_grid_apply(const SweepArgs &A, const double2 *__restrict__ side,
                                                  const double2 &e, double half) {
    using V_t = typename VT<D>::T;
    V_t *V = reinterpret_cast<V_t *>(A.V);
    const long long key = __double_as_longlong(e.x);
    if (key < 0) {
        const long long code = -2 - key;
        const int cnt = (int)(code & 0xff);
        if (cnt) group_solve_entries_acc<D>(side + (code >> 8), cnt, A.inv_m, half, GlobalV<D>{V});
        else visit_group<D, true>(A, code >> 8, half);
        return;
    }
    const int i = (int)(uint32_t)key, j = (int)(uint32_t)((unsigned long long)key >> 32);
    const double c = half * e.y;
    const double ca = c * __ldg(A.inv_m + i), cb = c * __ldg(A.inv_m + j);
    const double den = 1.0 + ca + cb;
    V_t vi = vldcg(V + i), vj = vldcg(V + j);
    double a[3], b[3];
    vget(vi, a);
    vget(vj, b);
#pragma unroll
    for (int m = 0; m < D; ++m) {
        const double u = (a[m] - b[m]) / den;
        a[m] -= ca * u;
        b[m] += cb * u;
    }
    vset(vi, a);
    vset(vj, b);
    vst(V + i, vi);
    vst(V + j, vj);
}

template <int D>
__global__ void __launch_bounds__(kSerialGridThreads)
    k_sweep_serial_grid(SweepArgs A, const double2 *__restrict__ ent, const double2 *__restrict__ side,
                        const int64_t *__restrict__ level_ptr, int64_t nlevels, unsigned long long *bar,
                        const Ctrl *ctrl) {
    if (ctrl->done) return;  // the same decision on every CTA
    const double half = 0.5 * ctrl->dt * ctrl->eta;
    const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t nth = (int64_t)gridDim.x * blockDim.x;
    const double2 none = make_double2(__longlong_as_double(-1ll), 0.0);
    unsigned long long target = 0;
    for (int pass = 0; pass < 2; ++pass) {
        auto level = [&](int64_t s) { return pass == 0 ? s : nlevels - 1 - s; };
        // this thread's first entry of a step (static data: prefetched one
        // step ahead, across the barrier)
        auto fetch = [&](int64_t s) {
            if (s >= nlevels) return none;
            const int64_t L = level(s), k = __ldg(level_ptr + L) + tid;
            return k < __ldg(level_ptr + L + 1) ? __ldg(ent + k) : none;
        };
        double2 nxt = fetch(0);
        for (int64_t s = 0; s < nlevels; ++s) {
            const double2 e = nxt;
            nxt = fetch(s + 1);
            if (__double_as_longlong(e.x) != -1ll) {
                serial_grid_apply<D>(A, side, e, half);
                const int64_t L = level(s), k1 = __ldg(level_ptr + L + 1);
                for (int64_t k = __ldg(level_ptr + L) + tid + nth; k < k1; k += nth)
                    serial_grid_apply<D>(A, side, __ldg(ent + k), half);
            }
            grid_barrier(bar, target);
        }
    }
}

// one colour phase: thread per task, groups in task order (dir>0) or
// reversed (dir<0)
template <int D>
__global__ void __launch_bounds__(128) k_sweep_colour(SweepArgs A, int64_t t0, int64_t t1, int dir,
                                                      const int64_t *__restrict__ task_ptr,
                                                      const Ctrl *ctrl) {
    const int64_t t = t0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= t1 || ctrl->done) return;
    const double half = 0.5 * ctrl->dt * ctrl->eta;
    const int64_t g0 = task_ptr[t], g1 = task_ptr[t + 1];
    if (dir > 0)
        for (int64_t g = g0; g < g1; ++g) visit_group<D>(A, g, half);
    else
        for (int64_t g = g1 - 1; g >= g0; --g) visit_group<D>(A, g, half);
}

// the level-ordered entries of the shared-memory serial sweep (setup, once;
// MTSPH_SERIAL_SMEM=0 keeps the global-memory kernel)
// Which reference-order kernel runs: the shared-memory one when velocities
// and level table fit (MTSPH_SERIAL_SMEM=0 disables it), else the multi-CTA
// one when a level averages more groups than one CTA has threads
// (MTSPH_SERIAL_GRID=0 disables it, 1 forces it), else the one-CTA global
// kernel.  All three are bit-identical.
template <int D> void build_serial_entries(NbhDev &nb, const SweepArgs &A, cudaStream_t s) {
    if (nb.sweep != 1) return;
    const int64_t ng = nb.level_groups.n;
    if (ng == 0) return;
    const char *env = getenv("MTSPH_SERIAL_SMEM");
    const char *genv = getenv("MTSPH_SERIAL_GRID");
    const bool smem = !(env && atoi(env) == 0) && serial_smem_bytes(nb.n, D, nb.nlevels) <= kSerialSmemMax;
    nb.serial_grid = 0;
    if (!smem) {
        const int gmode = genv ? atoi(genv) : -1;
        const double per_level = (double)ng / (double)std::max<int64_t>(nb.nlevels, 1);
        if (gmode == 1 || (gmode != 0 && per_level > 2.0 * kSerialGridThreads)) {
            int dev = 0, sms = 0, per = 0;
            MT_CUDA(cudaGetDevice(&dev));
            MT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            MT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sweep_serial_grid<D>,
                                                                  kSerialGridThreads, 0));
            // every CTA must be resident (grid barrier).  Two threads per group
            // of an average level, so that the fuller levels still give a
            // thread one entry (entries of one thread are dependent L2 round
            // trips), at most one CTA per SM (the barrier's cost grows with
            // the grid).  Measured on a 2 M slice (6469 levels): 24 CTAs
            // 67.3 ms per sweep, 48 52.0, 96 43.4, 148 43.3, 296 48.4.
            const int64_t want = (int64_t)std::ceil(2.0 * per_level / kSerialGridThreads);
            nb.serial_grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, std::min<int64_t>(sms, (int64_t)sms * std::max(per, 1))));
            if (const char *ce = getenv("MTSPH_SERIAL_GRID_CTAS"))  // tuning override (still all co-resident)
                nb.serial_grid = (int)std::max<int64_t>(1, std::min<int64_t>(atoi(ce), (int64_t)sms * std::max(per, 1)));
            nb.serial_bar.alloc(1);
        }
        if (!nb.serial_grid) return;
    } else {
        // the shared-memory opt-in is a per-device function attribute: set it
        // on every build (on the device this problem lives on)
        MT_CUDA(cudaFuncSetAttribute(k_sweep_serial_smem<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kSerialSmemMax));
    }
    // side-table offsets of the small groups, in level order
    std::vector<int64_t> lg(ng), gp(nb.ngroups + 1), off(ng, 0);
    nb.level_groups.download(lg.data(), ng, s);
    nb.gptr.download(gp.data(), nb.ngroups + 1, s);
    MT_CUDA(cudaStreamSynchronize(s));
    int64_t tot = 0;
    for (int64_t k = 0; k < ng; ++k) {
        const int64_t c = gp[lg[k] + 1] - gp[lg[k]];
        off[k] = tot;
        if (c > 1 && c <= kGroupMax) tot += c;
    }
    DBuf<int64_t> off_d;
    off_d.upload(off.data(), ng, s);
    nb.serial_ent.alloc(ng);
    nb.serial_side.alloc(std::max<int64_t>(tot, 1));
    k_serial_entries<D><<<(unsigned)((ng + 255) / 256), 256, 0, s>>>(A, nb.level_groups.p, ng, off_d.p,
                                                                     nb.serial_ent.p, nb.serial_side.p);
    MT_LAUNCH_CHECK();
    MT_CUDA(cudaStreamSynchronize(s));   // off_d is freed on return
}

// launch one full sweep on stream s; returns the number of kernel launches
template <int D>
int launch_sweep(const NbhDev &nb, const SweepArgs &A, const int64_t *level_ptr_d, const Ctrl *ctrl,
                 cudaStream_t s) {
    if (nb.npairs == 0) return 0;
    if (nb.sweep == 1) {
        const size_t sm = serial_smem_bytes(nb.n, D, nb.nlevels);
        if (nb.serial_grid > 0 && nb.serial_ent.n) {
            MT_CUDA(cudaMemsetAsync(nb.serial_bar.p, 0, sizeof(unsigned long long), s));
            k_sweep_serial_grid<D><<<(unsigned)nb.serial_grid, kSerialGridThreads, 0, s>>>(
                A, nb.serial_ent.p, nb.serial_side.p, level_ptr_d, nb.nlevels, nb.serial_bar.p, ctrl);
            MT_LAUNCH_CHECK();
            return 1;
        }
        if (nb.serial_ent.n && sm <= kSerialSmemMax) {
            k_sweep_serial_smem<D><<<1, kSerialThreads, sm, s>>>(A, nb.serial_ent.p, nb.serial_side.p, level_ptr_d,
                                                                 nb.nlevels, (int)nb.n, ctrl);
            MT_LAUNCH_CHECK();
            return 1;
        }
        k_sweep_serial<D><<<1, 1024, 0, s>>>(A, level_ptr_d, nb.nlevels, nb.level_groups.p, ctrl);
        MT_LAUNCH_CHECK();
        return 1;
    }
    int launches = 0;
    const int nc = (int)nb.colour_task_ptr.size() - 1;
    for (int pass = 0; pass < 2; ++pass)
        for (int q = 0; q < nc; ++q) {
            const int c = pass == 0 ? q : nc - 1 - q;
            const int64_t t0 = nb.colour_task_ptr[c], t1 = nb.colour_task_ptr[c + 1];
            if (t1 <= t0) continue;
            k_sweep_colour<D><<<blocks_for(t1 - t0, 128), 128, 0, s>>>(A, t0, t1, pass == 0 ? 1 : -1,
                                                                        nb.task_ptr.p, ctrl);
            MT_LAUNCH_CHECK();
            ++launches;
        }
    return launches;
}

}  // namespace mtsph
