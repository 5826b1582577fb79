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

// minimum resident CTAs per SM (register caps 85 / 64): measured at 10M (3D)
// with the chunked table, accel 5.28 ms at 3 CTAs, 5.23 at 4 (spills), 6.15
// at 2; stress (with the return map) 5.26 at 3, 5.06 at 4, 6.18 at 2
#ifndef MTSPH_STRESS_CTAS
#define MTSPH_STRESS_CTAS 4
#endif
// dF/dt gather: a test per visit (0) or unconditional visits per full word (1)
#ifndef MTSPH_STRESS_FAST
#define MTSPH_STRESS_FAST 0
#endif
#ifndef MTSPH_ACCEL_CTAS
#define MTSPH_ACCEL_CTAS 3
#endif
namespace mtsph {

// ---- chunked index table (C16 kernels) ----------------------------------
// With G lanes striding a row, each index load is 4 B per lane: G x 4 B per
// particle, one L1 wavefront per particle and iteration for 16 useful bytes
// -- 8 of the ~46 (dF/dt) / ~65 (divergence) wavefronts of a warp iteration
// with 4 lanes.  The chunked copy of the table stores every row in chunks of
// 4 G entries, permuted so lane l's next four entries (l, G + l, 2 G + l,
// 3 G + l of the chunk -- the entries it visits anyway, in the same order) are
// one 16 B word: one index wavefront per particle every four iterations.
// Rows are padded to whole chunks with -1: the full chunks run four
// unconditional visits, the row's last chunk tests each entry (walk_chunks).
__global__ void k_chunk_count(int64_t n, const int64_t *__restrict__ indptr, int g, int64_t *cnt) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i > n) return;
    cnt[i] = i < n ? (indptr[i + 1] - indptr[i] + 4 * g - 1) / (4 * g) : 0;
}
// One thread per particle.  pack: the row is first reordered so the four
// entries of every window (one 256-bit load of a 4-lane group) have
// distinct ids mod 4.  Measured (profiles/tools/l1_gather_ubench.cu): the L1
// returns a 4-lane group's four 32 B records in one cycle when their sector
// offsets within a 128 B line (id mod 4) differ, whatever lines they are in
// (a group straddling two lines: 8.5 cycles per warp load, as 8.2 aligned),
// and serialises equal offsets (four lines at one offset: 32 cycles; random
// records: 20).  A sorted row's windows break at cell boundaries: offline on
// the bench lattice 1.55 cycles per window, 1.15 after this reordering.
// Greedy and local: four queues by id mod 4 in ascending order, a window
// takes the head of every non-empty queue and fills up from the longest one
// (mean displacement ~4 entries, so a warp's eight rows still walk memory
// together).  Packing windows by whole 128 B lines instead (2.38 -> 1.97
// lines per window) measured no gain (stress 5.32 -> 5.36 ms, accel 5.64 ->
// 5.65): lines are not what the L1 data stage counts.
constexpr int kChunkMaxRow = 192;
__global__ void k_chunk_fill(int64_t n, const int64_t *__restrict__ indptr, const int32_t *__restrict__ csr, int g,
                             int pack, const int64_t *__restrict__ cptr, int32_t *out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t k0 = indptr[i];
    const int len = (int)(indptr[i + 1] - k0);
    const int64_t c0 = cptr[i], nch = cptr[i + 1] - c0;
    int32_t row[kChunkMaxRow];
    const bool packed = pack && len <= kChunkMaxRow;
    if (packed) {
        int cur[4], cnt[4] = {0, 0, 0, 0};
        for (int e = 0; e < len; ++e) ++cnt[csr[k0 + e] & 3];
        auto seek = [&](int k, int from) {
            while (from < len && (csr[k0 + from] & 3) != k) ++from;
            return from;
        };
        for (int k = 0; k < 4; ++k) cur[k] = seek(k, 0);
        int w = 0;
        while (w < len) {
            int32_t take[4];
            int m = 0;
            for (int k = 0; k < 4; ++k)
                if (cnt[k]) {
                    take[m++] = csr[k0 + cur[k]];
                    cur[k] = seek(k, cur[k] + 1);
                    --cnt[k];
                }
            while (m < 4 && w + m < len) {  // a queue ran dry: fill up from the longest one
                int k = 0;
                for (int q = 1; q < 4; ++q)
                    if (cnt[q] > cnt[k]) k = q;
                take[m++] = csr[k0 + cur[k]];
                cur[k] = seek(k, cur[k] + 1);
                --cnt[k];
            }
            for (int x = 1; x < m; ++x)  // ascending within the window
                for (int y = x; y > 0 && take[y] < take[y - 1]; --y) {
                    const int32_t t = take[y];
                    take[y] = take[y - 1];
                    take[y - 1] = t;
                }
            for (int x = 0; x < m; ++x) row[w++] = take[x];
        }
    }
    for (int64_t c = 0; c < nch; ++c)
        for (int l = 0; l < g; ++l) {
            int4 w;
            int32_t *wp = &w.x;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int64_t e = c * 4 * g + (int64_t)q * g + l;
                wp[q] = e < len ? (packed ? row[e] : csr[k0 + e]) : -1;
            }
            reinterpret_cast<int4 *>(out)[(c0 + c) * g + l] = w;
        }
}

// Per entry of the chunked table, the static magnitude factor of the kernel
// gradient, gradW_ab = mag_ab (X_b - X_a) / h^2 -- the one-time "precomputed
// kernel gradient" of the neighbour build in its cheapest form to stream
// (8 B per entry, a lane's next four in one 32 B word next to its four ids).
// Computed by grad_mag, the function the gathers would call: the stored
// gradient is bit-identical to the recomputed one.
template <int D>
__global__ void k_chunk_mag(int64_t n, const double4 *__restrict__ XV, KSpec ks, int g,
                            const int64_t *__restrict__ cptr, const int32_t *__restrict__ csr16, double *mag16) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    double xa[3];
    xget<D>(ldg4(XV + i), xa);
    const int64_t w0 = cptr[i] * g, w1 = cptr[i + 1] * g;
    for (int64_t w = w0; w < w1; ++w) {
        const int4 q = reinterpret_cast<const int4 *>(csr16)[w];
        const int32_t b[4] = {q.x, q.y, q.z, q.w};
        double m[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            m[e] = 0.0;
            if (b[e] >= 0) {
                double xb[3], rel[D], ww[D];
                xget<D>(ldg4(XV + b[e]), xb);
#pragma unroll
                for (int k = 0; k < D; ++k) rel[k] = xb[k] - xa[k];
                m[e] = grad_mag<D>(rel, ks, ww);
            }
        }
        reinterpret_cast<double4 *>(mag16)[w] = make_double4(m[0], m[1], m[2], m[3]);
    }
}

}  // namespace mtsph
namespace mtsph {
// build the chunked table for g lanes per particle (MTSPH_GATHER_CHUNKED=0: keep the CSR walk)
// (the solid's kernels have a CSR fallback; the porous ones need the table: required)
inline void build_chunked(NbhDev &nb, int g, cudaStream_t s, bool required = false, bool with_mag = false) {
    nb.chunk_g = 0;
    nb.mag16.release();
    if (const char *e = std::getenv("MTSPH_GATHER_CHUNKED"); !required && e && e[0] == '0') return;
    if (g < 2 || nb.n == 0) return;
    const int64_t n = nb.n;
    DBuf<int64_t> cnt((size_t)n + 1);
    k_chunk_count<<<blocks_for(n + 1), 256, 0, s>>>(n, nb.indptr.p, g, cnt.p);
    MT_LAUNCH_CHECK();
    nb.cptr.alloc((size_t)n + 1);
    CubTemp tmp;
    exclusive_scan(tmp, cnt.p, nb.cptr.p, n + 1, s);
    int64_t total = 0;
    MT_CUDA(cudaMemcpyAsync(&total, nb.cptr.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaStreamSynchronize(s));
    nb.csr16.alloc((size_t)total * 4 * g);
    // bank-balanced windows for 4 lanes per particle (MTSPH_GATHER_PACK=0: sorted rows)
    int pack = g == 4 ? 1 : 0;
    if (const char *e = std::getenv("MTSPH_GATHER_PACK")) pack = e[0] != '0' && g == 4;
    k_chunk_fill<<<blocks_for(n, 128), 128, 0, s>>>(n, nb.indptr.p, nb.csr.p, g, pack, nb.cptr.p, nb.csr16.p);
    MT_LAUNCH_CHECK();
    // stored kernel-gradient magnitudes (MTSPH_GATHER_MAG=0: recompute in the gathers)
    const char *me = std::getenv("MTSPH_GATHER_MAG");
    if (with_mag && (required || !(me && me[0] == '0'))) {
        nb.mag16.alloc((size_t)total * 4 * g);
        if (nb.d == 2) k_chunk_mag<2><<<blocks_for(n, 128), 128, 0, s>>>(n, nb.XV.p, nb.ks, g, nb.cptr.p, nb.csr16.p, nb.mag16.p);
        else k_chunk_mag<3><<<blocks_for(n, 128), 128, 0, s>>>(n, nb.XV.p, nb.ks, g, nb.cptr.p, nb.csr16.p, nb.mag16.p);
        MT_LAUNCH_CHECK();
    }
    MT_CUDA(cudaStreamSynchronize(s));
    nb.chunk_g = g;
}

// This lane's entries of particle i's row in the chunked table; visit(b, mag)
// with MAG (the stored gradient magnitudes next to the ids), else visit(b).
// MODE 0: a test per entry (padding is -1).  The dF/dt gathers run at a
//   tighter register cap (4 CTAs/SM in fp64), where an overlapped schedule
//   spills (6.25 vs 5.06 ms).
// MODE 1: four unconditional visits per full 16 B word -- the compiler
//   overlaps the next visit's loads with the current one's arithmetic -- and
//   tests in a partial word (the row's last few).  accel at 10M: 5.28 ms with
//   tests only, 5.27 so, 5.36 peeled, 5.18 with rows padded by the particle
//   itself (a zero contribution; no waste on the regular bar, ~10 % wasted
//   visits on rows of irregular length).
// MODE 2: peeled -- every chunk but the row's last unconditional, the last
//   one tested.  The register-heavy porous gathers: outer step (17 M plate)
//   33.2 ms peeled, 39.5 with MODE 1's two bodies in the loop, 37.1 CSR.
template <int G, int MODE, bool MAG, class F>
__device__ __forceinline__ void walk_chunks_any(const int64_t *__restrict__ cptr, const int32_t *__restrict__ csr16,
                                                const double *__restrict__ mag16, int64_t i, int sub, F &&visit) {
    const int64_t c0 = cptr[i];
    const int nch = (int)(cptr[i + 1] - c0);
    const int4 *w = reinterpret_cast<const int4 *>(csr16) + c0 * G + sub;
    const double4 *mw = reinterpret_cast<const double4 *>(mag16) + c0 * G + sub;
    auto call = [&](int32_t b, double m) {
        if constexpr (MAG) visit(b, m);
        else visit(b);
    };
    auto full = [&](const int4 &q, const double4 &m) {
        call(q.x, m.x);
        call(q.y, m.y);
        call(q.z, m.z);
        call(q.w, m.w);
    };
    auto tested = [&](const int4 &q, const double4 &m) {
        if (q.x >= 0) call(q.x, m.x);
        if (q.y >= 0) call(q.y, m.y);
        if (q.z >= 0) call(q.z, m.z);
        if (q.w >= 0) call(q.w, m.w);
    };
    const int nfull = MODE == 2 ? nch - 1 : nch;
    for (int c = 0; c < nfull; ++c, w += G, mw += G) {
        // the table words are a pure stream from DRAM, and a chunk's first
        // visit needs its word at once: hint them into L1 two chunks ahead
        // (stress 4.78 -> 4.68 ms, accel 5.27 -> 5.22; holding the next word
        // in registers instead spills, and prefetching the records the next
        // word names costs the data stage as much as loading them: 7.3 ms)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(w + 2 * G));
        if (MAG) asm volatile("prefetch.global.L1 [%0];" ::"l"(mw + 2 * G));
        const int4 q = __ldg(w);
        const double4 m = MAG ? ldg4(mw) : make_double4(0.0, 0.0, 0.0, 0.0);
        if (MODE == 2 || (MODE == 1 && q.w >= 0)) full(q, m);
        else tested(q, m);
    }
    if (MODE == 2 && nch > 0) {
        const int4 q = __ldg(w);
        const double4 m = MAG ? ldg4(mw) : make_double4(0.0, 0.0, 0.0, 0.0);
        tested(q, m);
    }
}
template <int G, bool FAST, class F>
__device__ __forceinline__ void walk_chunks(const int64_t *__restrict__ cptr, const int32_t *__restrict__ csr16,
                                            int64_t i, int sub, F &&visit) {
    walk_chunks_any<G, FAST ? 1 : 0, false>(cptr, csr16, nullptr, i, sub, visit);
}
template <int G, bool FAST, class F>
__device__ __forceinline__ void walk_chunks_mag(const int64_t *__restrict__ cptr, const int32_t *__restrict__ csr16,
                                                const double *__restrict__ mag16, int64_t i, int sub, F &&visit) {
    walk_chunks_any<G, FAST ? 1 : 0, true>(cptr, csr16, mag16, i, sub, visit);
}

template <int G, int K> __device__ __forceinline__ void group_sum(double (&v)[K]) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}

// dF/dt gather + F update (the split path: the return map runs in k_solid_rmap)
template <int D, int G, bool C16 = false, bool MAG = false, int TW = 1, int NP = 1>
__global__ void __launch_bounds__(256 * TW, TW == 1 ? MTSPH_STRESS_CTAS : 1) k_solid_stress_csr(SolidArgs A) {
    using V_t = typename VT<D>::T;
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const double dt = c->dt;
    const int64_t n = A.n;
    const int sub = threadIdx.x % G;
    const V_t *V = reinterpret_cast<const V_t *>(A.V);
    for (int it = 0; it < G * NP; ++it) {
        const int64_t i = (int64_t)blockIdx.x * (256 * TW * NP) + it * (256 * TW / G) + threadIdx.x / G;
        const bool act = i < n && !(A.flags[i] & FL_GHOST);  // uniform over the G lanes
        double acc[D * D];
#pragma unroll
        for (int k = 0; k < D * D; ++k) acc[k] = 0.0;
        if (act) {
            double xa[3], va[3];
            xget<D>(ldg4(A.XV + i), xa);
            vget(vldg(V + i), va);
            auto visit2 = [&](int32_t b, double mag) {
                const double4 xvb = ldg4(A.XV + b);
                double xb[3], vb[3], rel[D], g[D];
                xget<D>(xvb, xb);
                vget(vldg(V + b), vb);
#pragma unroll
                for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
                if (MAG) grad_w_mag<D>(rel, A.ks, mag, g);
                else grad_w<D>(rel, A.ks, g);
                const double volb = volof<D>(xvb);
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    const double dv = volb * (vb[r] - va[r]);
#pragma unroll
                    for (int cc = 0; cc < D; ++cc) acc[r * D + cc] += dv * g[cc];
                }
            };
            auto visit = [&](int32_t b) { visit2(b, 0.0); };
            if constexpr (C16 && MAG) {
                walk_chunks_mag<G, MTSPH_STRESS_FAST != 0>(A.cptr, A.csr16, A.mag16, i, sub, visit2);
            } else if constexpr (C16) {
                walk_chunks<G, MTSPH_STRESS_FAST != 0>(A.cptr, A.csr16, i, sub, visit);
            } else {
                const int64_t k1 = A.indptr[i + 1];
                for (int64_t k = A.indptr[i] + sub; k < k1; k += G) visit(__ldg(A.csr + k));
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
// TW: 1 = a 256-thread CTA works through its 256 particles 64 at a time (three
// such CTAs per SM, from blocks far apart); 3 = one 768-thread CTA per SM
// works through 768 particles 192 consecutive ones at a time, so the
// particles in flight on an SM are one compact neighbourhood in its L1
template <int D, int G, bool C16 = false, bool MAG = false, int TW = 1, int NP = 1>
__global__ void __launch_bounds__(256 * TW, TW == 1 ? MTSPH_ACCEL_CTAS : 1) k_solid_accel_csr(SolidArgs A) {
    using V_t = typename VT<D>::T;
    __shared__ double sh[32];
    const Ctrl *c = A.ctrl;
    if (c->done) return;  // uniform across the grid
    const double dt = c->dt;
    const int64_t n = A.n;
    const int sub = threadIdx.x % G;
    double ek = 0.0, a2m = 0.0;
    for (int it = 0; it < G * NP; ++it) {
        const int64_t i = (int64_t)blockIdx.x * (256 * TW * NP) + it * (256 * TW / G) + threadIdx.x / G;
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
            auto visit2 = [&](int32_t b, double mag) {
                double xb[3], Tb[D * D], rel[D], g[D];
                dload<D>(A.T, n, A.XV, b, Tb, xb);
#pragma unroll
                for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
                if (MAG) grad_w_mag<D>(rel, A.ks, mag, g);
                else grad_w<D>(rel, A.ks, g);
#pragma unroll
                for (int r = 0; r < D; ++r)
#pragma unroll
                    for (int cc = 0; cc < D; ++cc) acc[r] = fma(Tb[r * D + cc], g[cc], acc[r]);
            };
            auto visit = [&](int32_t b) { visit2(b, 0.0); };
            if constexpr (C16 && MAG) {
                walk_chunks_mag<G, true>(A.cptr, A.csr16, A.mag16, i, sub, visit2);
            } else if constexpr (C16) {
                walk_chunks<G, true>(A.cptr, A.csr16, i, sub, visit);
            } else {
                const int64_t k1 = A.indptr[i + 1];
                for (int64_t k = A.indptr[i] + sub; k < k1; k += G) visit(__ldg(A.csr + k));
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
    const double se = block_sum<256 * TW>(ek, sh);
    const double sa = block_max<256 * TW>(a2m, sh);
    // a wide CTA covers TW NP of the 256-particle blocks the partial rows are
    // laid out for: its sums go to the first of their slots, zeros to the rest
    // (the control kernel reduces all nblk slots)
    if (threadIdx.x < TW * NP) {
        const int64_t slot = (int64_t)blockIdx.x * (TW * NP) + threadIdx.x;
        if (slot < A.nblk) {
            A.part[slot] = threadIdx.x == 0 ? se : 0.0;
            A.part[A.nblk + slot] = threadIdx.x == 0 ? sa : 0.0;
        }
    }
}

}  // namespace mtsph
