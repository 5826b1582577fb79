// tgather.cuh -- block-tiled neighbour gathers (tiled pipeline).
//
// The two neighbour sums of the inner step -- the deformation-rate gather
// (solids.py:364) and the stress divergence (solids.py:416) -- read, for
// every particle, ~80 neighbours' reference positions and velocities or
// corrected stresses.  Gathering them straight from HBM through L1 is
// bound by L1 sector throughput (every warp load touches ~25 sectors).
// Here one CTA serves one Morton block of cells (the blocks of the tiled
// damping sweep): it stages the block's halo (the block grown by one cell,
// a union of contiguous cell ranges) into shared memory with coalesced
// loads, then every owned particle sums over its neighbours through a
// 16-bit block-local neighbour table.  Sums run in the same neighbour
// order as the SELL kernels, so results are identical to round-off.
#pragma once

#include "solid.cuh"
#include "tiled.cuh"

namespace mtsph {

struct GatherArgs {
    const int64_t *range_off;
    const int2 *ranges;
    const int32_t *halo_n;
    const int64_t *nl_off, *self_off;
    const uint16_t *nl, *self;
    const int32_t *width, *own0, *own_n;
};

inline GatherArgs gather_args(const TiledSched &t) {
    return GatherArgs{t.range_off.p, t.ranges.p, t.halo_n.p, t.nl_off.p, t.self_off.p,
                      t.nl.p, t.self.p, t.width.p, t.own0.p, t.own_n.p};
}

// shared-memory range table + global index of local halo slot l
struct HaloMap {
    const int2 *rt;
    int nr;
    __device__ __forceinline__ int64_t global(int l) const {
        int lo = 0, hi = nr - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (rt[mid].y <= l) lo = mid; else hi = mid - 1;
        }
        return (int64_t)rt[lo].x + (l - rt[lo].y);
    }
};

__device__ __forceinline__ HaloMap stage_ranges(const GatherArgs &G, int64_t task, double *smem, int &H,
                                                double *&rest) {
    const int64_t r0 = G.range_off[task], r1 = G.range_off[task + 1];
    const int nr = (int)(r1 - r0);
    int2 *rt = reinterpret_cast<int2 *>(smem);
    for (int r = threadIdx.x; r < nr; r += blockDim.x) rt[r] = G.ranges[r0 + r];
    H = G.halo_n[task];
    rest = smem + (((nr + 1) & ~1) + 3) / 4 * 4;
    return HaloMap{rt, nr};
}

inline size_t gather_smem_bytes(const TiledSched &t, int per_particle_doubles) {
    return (size_t)((((t.max_ranges + 1) & ~1) + 3) / 4 * 4) * 8 +
           (size_t)t.max_halo * per_particle_doubles * 8;
}

// dF/dt gather + F update for the owned particles of one block
template <int D>
__global__ void __launch_bounds__(256) k_stress_tiled(SolidArgs A, GatherArgs G) {
    using V_t = typename VT<D>::T;
    extern __shared__ double smem[];
    if (A.ctrl->done) return;
    const int64_t task = blockIdx.x;
    int H;
    double *rest;
    const HaloMap hm = stage_ranges(G, task, smem, H, rest);
    double4 *sx = reinterpret_cast<double4 *>(rest);       // X | vol
    double4 *sv = sx + H;                                   // v (padded)
    __syncthreads();
    const V_t *V = reinterpret_cast<const V_t *>(A.V);
    for (int l = threadIdx.x; l < H; l += blockDim.x) {
        const int64_t g = hm.global(l);
        sx[l] = ldg4(A.XV + g);
        double v[3] = {0, 0, 0};
        vget(V[g], v);
        sv[l] = make_double4(v[0], v[1], v[2], 0.0);
    }
    __syncthreads();
    const double dt = A.ctrl->dt;
    const int64_t n = A.n;
    const int cnt = G.own_n[task], W = G.width[task];
    const int64_t nb = G.nl_off[task], sb = G.self_off[task];
    const int64_t a0 = G.own0[task];
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
        const int64_t i = a0 + k;
        const int sl = G.self[sb + k];
        const double4 xa4 = sx[sl], va4 = sv[sl];
        const double xa[3] = {xa4.x, xa4.y, xa4.z}, va[3] = {va4.x, va4.y, va4.z};
        double acc[D * D];
#pragma unroll
        for (int q = 0; q < D * D; ++q) acc[q] = 0.0;
        for (int m = 0; m < W; ++m) {
            const int l = G.nl[nb + (int64_t)m * cnt + k];
            const double4 xb4 = sx[l], vb4 = sv[l];
            const double xb[3] = {xb4.x, xb4.y, xb4.z}, vb[3] = {vb4.x, vb4.y, vb4.z};
            double rel[D], g[D];
#pragma unroll
            for (int c = 0; c < D; ++c) rel[c] = xb[c] - xa[c];
            grad_w<D>(rel, A.ks, g);
            const double volb = volof<D>(xb4);
#pragma unroll
            for (int r = 0; r < D; ++r) {
                const double dv = volb * (vb[r] - va[r]);
#pragma unroll
                for (int c = 0; c < D; ++c) acc[r * D + c] += dv * g[c];
            }
        }
        double Bm[D * D], L[D * D];
#pragma unroll
        for (int q = 0; q < D * D; ++q) Bm[q] = A.B[(int64_t)q * n + i];
        mm<D>(acc, Bm, L);
#pragma unroll
        for (int q = 0; q < D * D; ++q) A.F[(int64_t)q * n + i] += dt * L[q];
    }
}

// stress divergence + kick + energy / |a| partials (one per block)
template <int D>
__global__ void __launch_bounds__(256) k_accel_tiled(SolidArgs A, GatherArgs G) {
    using V_t = typename VT<D>::T;
    extern __shared__ double smem[];
    __shared__ double red[32];
    if (A.ctrl->done) return;
    const int64_t task = blockIdx.x;
    int H;
    double *rest;
    const HaloMap hm = stage_ranges(G, task, smem, H, rest);
    double4 *sx = reinterpret_cast<double4 *>(rest);       // X | vol
    double *sT = reinterpret_cast<double *>(sx + H);       // D*D per particle
    __syncthreads();
    for (int l = threadIdx.x; l < H; l += blockDim.x) {
        const int64_t g = hm.global(l);
        sx[l] = ldg4(A.XV + g);
        double t[D * D];
        tload<D>(A.T, A.n, g, t);
#pragma unroll
        for (int q = 0; q < D * D; ++q) sT[(size_t)l * D * D + q] = t[q];
    }
    __syncthreads();
    const double dt = A.ctrl->dt;
    const int64_t n = A.n;
    const int cnt = G.own_n[task], W = G.width[task];
    const int64_t nb = G.nl_off[task], sb = G.self_off[task];
    const int64_t a0 = G.own0[task];
    double ek = 0.0, a2m = 0.0;
    for (int k = threadIdx.x; k < cnt; k += blockDim.x) {
        const int64_t i = a0 + k;
        const int sl = G.self[sb + k];
        const double4 xa4 = sx[sl];
        const double xa[3] = {xa4.x, xa4.y, xa4.z};
        double Ta[D * D], acc[D];
#pragma unroll
        for (int q = 0; q < D * D; ++q) Ta[q] = sT[(size_t)sl * D * D + q];
#pragma unroll
        for (int c = 0; c < D; ++c) acc[c] = 0.0;
        for (int m = 0; m < W; ++m) {
            const int l = G.nl[nb + (int64_t)m * cnt + k];
            const double4 xb4 = sx[l];
            const double xb[3] = {xb4.x, xb4.y, xb4.z};
            const double *Tb = sT + (size_t)l * D * D;
            double rel[D], g[D];
#pragma unroll
            for (int c = 0; c < D; ++c) rel[c] = xb[c] - xa[c];
            grad_w<D>(rel, A.ks, g);
            const double volb = volof<D>(xb4);
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) s += (Ta[r * D + c] + Tb[r * D + c]) * g[c];
                acc[r] += volb * s;
            }
        }
        const double rho0 = A.rho0[i];
#pragma unroll
        for (int c = 0; c < D; ++c) {
            acc[c] /= rho0;
            A.a[(int64_t)c * n + i] = acc[c];
        }
        if (A.flags[i] & FL_MOVABLE) {
            V_t *V = reinterpret_cast<V_t *>(A.V);
            double v[3];
            vget(V[i], v);
            double v2 = 0.0, aa = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                v[c] += 0.5 * dt * acc[c];
                v2 += v[c] * v[c];
                aa += acc[c] * acc[c];
            }
            V_t w;
            vset(w, v);
            V[i] = w;
            ek += A.mass[i] * v2;
            a2m = fmax(a2m, aa);
        }
    }
    const double se = block_sum<256>(ek, red);
    const double sa = block_max<256>(a2m, red);
    if (threadIdx.x == 0) {
        A.part[task] = se;
        A.part[A.nblk + task] = sa;
    }
}

}  // namespace mtsph
