// gather_csr.cuh -- row-parallel neighbour gathers (G lanes per particle).
//
// The SELL gathers (solid.cuh) give each lane one particle and step all 32
// lanes through their m-th neighbours: 32 particles' m-th neighbours are
// ~23 different records on as many cache lines, and the L1 data stage (one
// wavefront per line a warp load touches) is the bound.  Here G lanes share
// one particle and walk its sorted CSR row with stride G: consecutive entries
// of a sorted row are mostly consecutive particles of one neighbour cell, so
// a warp load touches 32/G particles x ~2 lines.  The G partial sums are
// combined with a fixed xor-shuffle tree (deterministic; the summation order
// differs from the SELL path by rounding only).
//
// Grid and partials layout are those of the SELL kernels (blocks of 256
// particles): a block loops over its particles 256/G at a time.
#pragma once

#include "solid.cuh"

// minimum resident CTAs per SM (register caps 85): measured at 10M (3D) accel
// 7.3 ms at 2 CTAs (92 regs), 6.3 ms at 3, 7.0 ms at 4 (spills); stress is
// flat from 3 up, and slower when the cap is lifted (1: 7.2 vs 5.8 ms)
#ifndef MTSPH_STRESS_CTAS
#define MTSPH_STRESS_CTAS 3
#endif
#ifndef MTSPH_ACCEL_CTAS
#define MTSPH_ACCEL_CTAS 3
#endif

namespace mtsph {

template <int G, int K> __device__ __forceinline__ void group_sum(double (&v)[K]) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}

// dF/dt gather + F update (the split path: the return map runs in k_solid_rmap)
template <int D, int G>
__global__ void __launch_bounds__(256, MTSPH_STRESS_CTAS) k_solid_stress_csr(SolidArgs A) {
    using V_t = typename VT<D>::T;
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const double dt = c->dt;
    const int64_t n = A.n;
    const int sub = threadIdx.x % G;
    const V_t *V = reinterpret_cast<const V_t *>(A.V);
    for (int it = 0; it < G; ++it) {
        const int64_t i = (int64_t)blockIdx.x * 256 + it * (256 / G) + threadIdx.x / G;
        const bool act = i < n && !(A.flags[i] & FL_GHOST);  // uniform over the G lanes
        double acc[D * D];
#pragma unroll
        for (int k = 0; k < D * D; ++k) acc[k] = 0.0;
        if (act) {
            double xa[3], va[3];
            xget<D>(ldg4(A.XV + i), xa);
            vget(vldg(V + i), va);
            const int64_t k1 = A.indptr[i + 1];
            for (int64_t k = A.indptr[i] + sub; k < k1; k += G) {
                const int32_t b = __ldg(A.csr + k);
                const double4 xvb = ldg4(A.XV + b);
                double xb[3], vb[3], rel[D], g[D];
                xget<D>(xvb, xb);
                vget(vldg(V + b), vb);
#pragma unroll
                for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
                grad_w<D>(rel, A.ks, g);
                const double volb = volof<D>(xvb);
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    const double dv = volb * (vb[r] - va[r]);
#pragma unroll
                    for (int cc = 0; cc < D; ++cc) acc[r * D + cc] += dv * g[cc];
                }
            }
        }
        group_sum<G>(acc);
        if (act && sub == 0) {
            double Bm[D * D], F[D * D], L[D * D];
#pragma unroll
            for (int k = 0; k < D * D; ++k) {
                Bm[k] = A.B[(int64_t)k * n + i];
                F[k] = A.F[(int64_t)k * n + i];
            }
            mm<D>(acc, Bm, L);
#pragma unroll
            for (int k = 0; k < D * D; ++k) A.F[(int64_t)k * n + i] = F[k] + dt * L[k];
        }
    }
}

// a = 1/rho0 sum_b V_b (T_a + T_b) gradW, v += dt/2 a, E_k and |a|max partials
template <int D, int G>
__global__ void __launch_bounds__(256, MTSPH_ACCEL_CTAS) k_solid_accel_csr(SolidArgs A) {
    using V_t = typename VT<D>::T;
    __shared__ double sh[32];
    const Ctrl *c = A.ctrl;
    if (c->done) return;  // uniform across the grid
    const double dt = c->dt;
    const int64_t n = A.n;
    const int sub = threadIdx.x % G;
    double ek = 0.0, a2m = 0.0;
    for (int it = 0; it < G; ++it) {
        const int64_t i = (int64_t)blockIdx.x * 256 + it * (256 / G) + threadIdx.x / G;
        const bool act = i < n && !(A.flags[i] & FL_GHOST);
        // sum_b V_b (T_a + T_b) gradW = sum_b T~_b gradW + T_a G_a, with
        // T~_b = V_b T_b from the divergence record (three 256-bit loads per
        // neighbour, X included) and G_a = sum_b V_b gradW static
        double acc[D];
#pragma unroll
        for (int k = 0; k < D; ++k) acc[k] = 0.0;
        if (act) {
            double xa[3];
            xget<D>(ldg4(A.XV + i), xa);
            const int64_t k1 = A.indptr[i + 1];
            for (int64_t k = A.indptr[i] + sub; k < k1; k += G) {
                const int32_t b = __ldg(A.csr + k);
                double xb[3], Tb[D * D], rel[D], g[D];
                dload<D>(A.T, n, A.XV, b, Tb, xb);
#pragma unroll
                for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
                grad_w<D>(rel, A.ks, g);
#pragma unroll
                for (int r = 0; r < D; ++r)
#pragma unroll
                    for (int cc = 0; cc < D; ++cc) acc[r] = fma(Tb[r * D + cc], g[cc], acc[r]);
            }
        }
        group_sum<G>(acc);
        if (act && sub == 0) {
            double Ta[D * D], xd[3];
            dload<D>(A.T, n, A.XV, i, Ta, xd);
            const double rho0 = A.rho0[i], vola = volof<D>(ldg4(A.XV + i));
#pragma unroll
            for (int k = 0; k < D; ++k) {
                double ta = 0.0;
#pragma unroll
                for (int cc = 0; cc < D; ++cc) ta += Ta[k * D + cc] * A.G[(int64_t)cc * n + i];
                acc[k] = (acc[k] + ta / vola) / rho0;
                A.a[(int64_t)k * n + i] = acc[k];
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
                ek += A.mass[i] * v2;
                a2m = fmax(a2m, aa);
            }
        }
    }
    const double se = block_sum<256>(ek, sh);
    const double sa = block_max<256>(a2m, sh);
    if (threadIdx.x == 0) {
        A.part[blockIdx.x] = se;
        A.part[A.nblk + blockIdx.x] = sa;
    }
}

}  // namespace mtsph
