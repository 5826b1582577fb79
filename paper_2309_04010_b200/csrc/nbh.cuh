// nbh.cuh -- one-time neighbourhood build on the GPU.
//
// Replaces neighbors.py:59 build_neighborhoods + neighbors.py:232
// compute_correction_matrices.  Steps (all on the device except O(#cells)
// scalar bookkeeping):
//   1. particles binned into cells of edge 2 in the scaled space u = X/h
//      (= the kernel support), sorted by Morton code of the cell (CUB
//      radix sort, stable -> original order inside a cell); this Morton
//      order is the internal particle order of every device array;
//   2. candidates from the 3^d neighbouring cells, accepted with the
//      reference's exact test |u_j - u_i| < 2 (IEEE ops in the reference's
//      order, so the neighbour SETS are bit-identical);
//   3. CSR (internal numbering, neighbours ascending) + a SELL-32 copy
//      (slices of 32 consecutive particles, column-major, padded with the
//      particle itself) for the coalesced thread-per-particle gathers;
//   4. correction matrices B = M^-1, M = sum_b V_b (X_b-X_a) (x) grad W;
//   5. the damping pair schedule: unique pairs (i < j in ORIGINAL ids, as
//      the reference) sorted with stable radix sorts that reproduce the
//      reference's np.lexsort keys (neighbors.py:96-108), equal-key runs
//      split into particle-sharing groups (neighbors.py:165), then either
//        SERIAL:   the reference order, level-scheduled (groups of one
//                  level touch disjoint particles) -> bit-exact sweep, or
//        COLOURED: the same keys below a (colour, task) prefix: midpoint
//                  cells of edge h, colour = (|c_k| mod 3)_k, so tasks of
//                  one colour never share a particle and run in parallel.
#pragma once

#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"

namespace mtsph {

struct CubTemp {
    DBuf<unsigned char> buf;
    void *ensure(size_t bytes) {
        if (bytes > buf.n) buf.alloc(bytes + (bytes >> 2) + 256);
        return buf.p;
    }
};

template <class K, class V>
void sort_pairs(CubTemp &tmp, const K *kin, K *kout, const V *vin, V *vout, int64_t n,
                int end_bit, cudaStream_t s) {
    size_t bytes = 0;
    MT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0,
                                            end_bit, s));
    void *t = tmp.ensure(bytes);
    MT_CUDA(cub::DeviceRadixSort::SortPairs(t, bytes, kin, kout, vin, vout, n, 0, end_bit, s));
}

template <class T>
void exclusive_scan(CubTemp &tmp, const T *in, T *out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    MT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    void *t = tmp.ensure(bytes);
    MT_CUDA(cub::DeviceScan::ExclusiveSum(t, bytes, in, out, n, s));
}

// ------------------------------------------------------------ device data

struct NbhDev {
    int64_t n = 0;
    int d = 0;
    KSpec ks{};
    double h_axes[3] = {1, 1, 1};
    double center[3] = {0, 0, 0};
    DBuf<int64_t> perm, iperm;   // internal -> original, original -> internal
    DBuf<double4> XV;            // (X, vol) internal order; X padded with 0
    // neighbour table
    int64_t nnz = 0;             // directed entries (2 * pairs)
    DBuf<int64_t> indptr;        // CSR over internal ids
    DBuf<int32_t> csr;
    // chunked copy for the row-parallel gathers (gather_csr.cuh build_chunked):
    // chunk offsets per particle and the permuted, padded entries
    int chunk_g = 0;             // lanes per particle it was built for (0: none)
    DBuf<int64_t> cptr;
    DBuf<int32_t> csr16;
    DBuf<double> mag16;          // per entry of csr16: the kernel-gradient magnitude factor (0 for padding)
    bool want_sell = false;      // SELL-32 only for the opt-in one-lane gathers
    int64_t nslices = 0, sell_size = 0;
    DBuf<int64_t> slice_ptr;
    DBuf<int32_t> slice_w;
    DBuf<int32_t> nbr;           // SELL-32
    DBuf<double> B;              // corrections SoA [d*d][n]
    // pair schedule
    int sweep = 0;
    DBuf<uint64_t> cellkey;      // sorted Morton cell key per particle
    bool has_grid = false;       // global cell grid (multi-rank), scaled space
    double grid_lo[3] = {0, 0, 0}, grid_hi[3] = {0, 0, 0};
    std::vector<uint8_t> ghost_internal;  // 1 = ghost (internal order), empty = none
    const uint8_t *ghost_orig = nullptr;  // during the build: ghost flags, caller order
                                          // (ghosts may have one-sided, singular moments)
    int64_t npairs = 0, ngroups = 0;
    DBuf<int32_t> pi, pj;        // internal ids, reference orientation
    DBuf<int64_t> gptr;          // group -> pair range
    DBuf<int64_t> gscr;          // group scratch offset (doubles), -1 single
    int64_t scratch_doubles = 0;
    DBuf<double> scratch;
    // SERIAL
    int64_t nlevels = 0;
    std::vector<int64_t> level_ptr_h;
    DBuf<int64_t> level_groups;
    DBuf<double2> serial_ent;    // level-ordered sweep entries (damping.cuh k_serial_entries)
    DBuf<double2> serial_side;   // pair entries of the small simultaneous-solve groups
    int serial_grid = 0;         // CTAs of the multi-CTA serial kernel (0: not used)
    DBuf<unsigned long long> serial_bar;  // its grid barrier (monotonic arrivals, zeroed per launch)
    // COLOURED: phases (colours) -> tasks -> groups
    std::vector<int64_t> colour_task_ptr;  // ncolours+1 over tasks
    DBuf<int64_t> task_ptr;                // ntasks+1 over groups
    int64_t ntasks = 0;
};

// ------------------------------------------------------------ kernels

template <int D>
__global__ void k_cell_keys(int64_t n, const double *__restrict__ pos, KSpec ks, double3 lo,
                            int3 dims, uint64_t *key, int64_t *val) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double lov[3] = {lo.x, lo.y, lo.z};
    const int dv[3] = {dims.x, dims.y, dims.z};
    uint64_t c[3] = {0, 0, 0};
#pragma unroll
    for (int k = 0; k < D; ++k) {
        // u = x / h exactly as the reference (IEEE division)
        double u = __ddiv_rn(pos[i * D + k], ks.h[k]);
        int64_t ck = (int64_t)floor((u - lov[k]) * 0.5);
        ck = ck < 0 ? 0 : (ck >= dv[k] ? dv[k] - 1 : ck);
        c[k] = (uint64_t)ck;
    }
    key[i] = (D == 3) ? (spread3(c[0]) | spread3(c[1]) << 1 | spread3(c[2]) << 2)
                      : (spread2(c[0]) | spread2(c[1]) << 1);
    val[i] = i;
}

template <int D>
__global__ void k_gather_sorted(int64_t n, const int64_t *__restrict__ perm,
                                const double *__restrict__ pos, const double *__restrict__ vol,
                                KSpec ks, int64_t *iperm, double4 *XV, double4 *U) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    int64_t o = perm[k];
    iperm[o] = k;
    double x[3] = {0, 0, 0}, u[3] = {0, 0, 0};
#pragma unroll
    for (int c = 0; c < D; ++c) {
        x[c] = pos[o * D + c];
        u[c] = __ddiv_rn(x[c], ks.h[c]);
    }
    XV[k] = D == 3 ? make_double4(x[0], x[1], x[2], vol[o]) : make_double4(x[0], x[1], vol[o], 0.0);
    U[k] = make_double4(u[0], u[1], u[2], 0.0);
}

__global__ void k_cell_starts(int64_t n, const uint64_t *__restrict__ key, int64_t *flag) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    flag[k] = (k == 0 || key[k] != key[k - 1]) ? 1 : 0;
}

__global__ void k_cell_index(int64_t n, const int64_t *__restrict__ flag,
                             const int64_t *__restrict__ scan, int64_t *cell_of,
                             int64_t *cell_start, uint64_t *cell_key, const uint64_t *key) {
    int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    int64_t c = scan[k] + flag[k] - 1;
    cell_of[k] = c;
    if (flag[k]) { cell_start[c] = k; cell_key[c] = key[k]; }
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t *a, int64_t n, uint64_t x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// for each occupied cell: indices of its (up to 3^d) occupied neighbour
// cells, ascending by Morton key (=> ascending internal particle ids)
template <int D>
__global__ void k_cell_neighbours(int64_t ncell, const uint64_t *__restrict__ cell_key,
                                  int3 dims, int32_t *cnb /* ncell x 27 */) {
    int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= ncell) return;
    uint64_t key = cell_key[c];
    int64_t cc[3] = {0, 0, 0};
    // de-interleave
#pragma unroll
    for (int k = 0; k < D; ++k) {
        uint64_t v = 0;
        for (int b = 0; b < (D == 3 ? 21 : 32); ++b) v |= ((key >> (b * D + k)) & 1ull) << b;
        cc[k] = (int64_t)v;
    }
    const int dv[3] = {dims.x, dims.y, dims.z};
    uint64_t keys[27];
    int m = 0;
    for (int o2 = (D == 3 ? -1 : 0); o2 <= (D == 3 ? 1 : 0); ++o2)
        for (int o1 = -1; o1 <= 1; ++o1)
            for (int o0 = -1; o0 <= 1; ++o0) {
                int64_t q[3] = {cc[0] + o0, cc[1] + o1, cc[2] + o2};
                bool ok = true;
                for (int k = 0; k < D; ++k) ok = ok && q[k] >= 0 && q[k] < dv[k];
                if (!ok) continue;
                keys[m++] = D == 3 ? (spread3(q[0]) | spread3(q[1]) << 1 | spread3(q[2]) << 2)
                                   : (spread2(q[0]) | spread2(q[1]) << 1);
            }
    // insertion sort ascending
    for (int a = 1; a < m; ++a) {
        uint64_t v = keys[a];
        int b = a - 1;
        while (b >= 0 && keys[b] > v) { keys[b + 1] = keys[b]; --b; }
        keys[b + 1] = v;
    }
    int w = 0;
    for (int a = 0; a < m; ++a) {
        int64_t idx = lower_bound_u64(cell_key, ncell, keys[a]);
        if (idx < ncell && cell_key[idx] == keys[a]) cnb[c * 27 + w++] = (int32_t)idx;
    }
    for (; w < 27; ++w) cnb[c * 27 + w] = -1;
}

// exact reference distance test in the scaled space (neighbors.py:82-90)
template <int D>
__device__ __forceinline__ double scaled_dist(const double4 &ui, const double4 &uj) {
    double d0 = __dsub_rn(uj.x, ui.x);
    double s = __dmul_rn(d0, d0);
    if (D >= 2) { double d1 = __dsub_rn(uj.y, ui.y); s = __dadd_rn(s, __dmul_rn(d1, d1)); }
    if (D >= 3) { double d2 = __dsub_rn(uj.z, ui.z); s = __dadd_rn(s, __dmul_rn(d2, d2)); }
    return __dsqrt_rn(s);
}

template <int D, bool FILL>
__global__ void k_neigh(int64_t n, const double4 *__restrict__ U, const int64_t *__restrict__ cell_of,
                        const int64_t *__restrict__ cell_start, int64_t ncell,
                        const int32_t *__restrict__ cnb, const int64_t *__restrict__ perm,
                        int64_t *count, const int64_t *__restrict__ indptr, int32_t *csr,
                        unsigned long long *dup) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double4 ui = U[i];
    const int64_t c = cell_of[i];
    int64_t cnt = 0;
    int64_t w = FILL ? indptr[i] : 0;
    for (int t = 0; t < 27; ++t) {
        int32_t cn = cnb[c * 27 + t];
        if (cn < 0) break;
        int64_t s0 = cell_start[cn], s1 = (cn + 1 < ncell) ? cell_start[cn + 1] : n;
        for (int64_t j = s0; j < s1; ++j) {
            if (j == i) continue;
            double q = scaled_dist<D>(ui, U[j]);
            if (q == 0.0) {
                if (!FILL) {
                    int64_t a = perm[i], b = perm[j];
                    unsigned long long lo = (unsigned long long)(a < b ? a : b);
                    atomicMin(dup, lo);
                }
                continue;
            }
            if (q < 2.0) {
                if (FILL) csr[w++] = (int32_t)j;
                ++cnt;
            }
        }
    }
    if (!FILL) count[i] = cnt;
}

__global__ void k_slice_width(int64_t n, int64_t nslices, const int64_t *__restrict__ count,
                              int32_t *slice_w, int64_t *slice_sz) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= nslices) return;
    int64_t w = 0;
    for (int l = 0; l < 32; ++l) {
        int64_t a = s * 32 + l;
        if (a < n && count[a] > w) w = count[a];
    }
    slice_w[s] = (int32_t)w;
    slice_sz[s] = w * 32;
}

__global__ void k_fill_sell(int64_t n, const int64_t *__restrict__ indptr,
                            const int32_t *__restrict__ csr, const int64_t *__restrict__ slice_ptr,
                            const int32_t *__restrict__ slice_w, int32_t *nbr) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t s = a >> 5;
    int l = (int)(a & 31);
    if (s * 32 >= n) return;
    int64_t base = slice_ptr[s];
    int w = slice_w[s];
    int64_t k0 = a < n ? indptr[a] : 0, k1 = a < n ? indptr[a + 1] : 0;
    for (int m = 0; m < w; ++m) {
        int64_t k = k0 + m;
        nbr[base + (int64_t)m * 32 + l] = (k < k1) ? csr[k] : (int32_t)(a < n ? a : 0);
    }
}

// correction matrices (neighbors.py:220-246); flags singular particles
template <int D>
__global__ void k_corrections(int64_t n, const double4 *__restrict__ XV, const int64_t *__restrict__ indptr,
                              const int32_t *__restrict__ csr, KSpec ks, double *B,
                              uint8_t *singular) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    const double4 xa = XV[a];
    const double xa_[3] = {xa.x, xa.y, xa.z};
    double M[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) M[k] = 0.0;
    for (int64_t k = indptr[a]; k < indptr[a + 1]; ++k) {
        const double4 xb = XV[csr[k]];
        const double xb_[3] = {xb.x, xb.y, xb.z};
        const double vb = D == 3 ? xb.w : xb.z;
        double rel[D], g[D];
        double r2 = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) { rel[c] = xb_[c] - xa_[c]; r2 += rel[c] * rel[c]; }
        const double r = sqrt(r2);
        grad_w<D>(rel, ks, g);
#pragma unroll
        for (int r0 = 0; r0 < D; ++r0) {
            const double relr = r * (rel[r0] / r);  // reference uses |r| * e
#pragma unroll
            for (int c = 0; c < D; ++c) M[r0 * D + c] += vb * relr * g[c];
        }
    }
    const double j = det_d<D>(M);
    double fro = 0.0;
#pragma unroll
    for (int k = 0; k < D * D; ++k) fro += M[k] * M[k];
    fro = sqrt(fro);
    double scale = fro;
    for (int k = 1; k < D; ++k) scale *= fro;
    scale += 2.2250738585072014e-308;
    double inv[D * D];
    const bool bad = !(fabs(j) > 1e-12 * scale);
    singular[a] = bad ? 1 : 0;
    if (!bad) inv_d<D>(M, j, inv);
#pragma unroll
    for (int k = 0; k < D * D; ++k) B[(int64_t)k * n + a] = bad ? 0.0 : inv[k];
}

// unique pairs from the CSR: a owns (a, b) when orig(a) < orig(b)
__global__ void k_pair_count(int64_t n, const int64_t *__restrict__ indptr, const int32_t *__restrict__ csr,
                             const int64_t *__restrict__ perm, int64_t *cnt) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    int64_t oa = perm[a], c = 0;
    for (int64_t k = indptr[a]; k < indptr[a + 1]; ++k) c += perm[csr[k]] > oa;
    cnt[a] = c;
}
__global__ void k_pair_fill(int64_t n, const int64_t *__restrict__ indptr, const int32_t *__restrict__ csr,
                            const int64_t *__restrict__ perm, const int64_t *__restrict__ off,
                            int32_t *pi, int32_t *pj) {
    int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    int64_t oa = perm[a], w = off[a];
    for (int64_t k = indptr[a]; k < indptr[a + 1]; ++k)
        if (perm[csr[k]] > oa) { pi[w] = (int32_t)a; pj[w] = csr[k]; ++w; }
}

__global__ void k_iota(int64_t n, uint32_t *p) {
    int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m < n) p[m] = (uint32_t)m;
}

// key of pair P[m] for sort pass `which` (see build_schedule)
template <int D>
__global__ void k_pair_key(int64_t np, const uint32_t *__restrict__ P, const int32_t *__restrict__ pi,
                           const int32_t *__restrict__ pj, const int64_t *__restrict__ perm,
                           const double4 *__restrict__ XV, double3 center, KSpec ks, int which,
                           uint64_t *key) {
    int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= np) return;
    const uint32_t p = P[m];
    const int32_t i = pi[p], j = pj[p];
    uint64_t out = 0;
    if (which == 0) out = (uint64_t)perm[j];
    else if (which == 1) out = (uint64_t)perm[i];
    else {
        const double4 a = XV[i], b = XV[j];
        const double ca[3] = {a.x, a.y, a.z}, cb[3] = {b.x, b.y, b.z};
        const double cen[3] = {center.x, center.y, center.z};
        double cm[3];
#pragma unroll
        for (int k = 0; k < D; ++k) cm[k] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(ca[k], cb[k])), cen[k]);
        if (which >= 2 && which < 2 + D) out = dkey(cm[D - 1 - (which - 2)]);
        else if (which >= 2 + D && which < 2 + 2 * D) out = dkey(fabs(cm[D - 1 - (which - 2 - D)]));
        else {
            // colour / task of the midpoint cell (edge h, centred, symmetric rounding)
            int64_t t[3] = {0, 0, 0};
            int col = 0, mul = 1;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                double x = cm[k] * ks.inv_h[k];
                int64_t c = (int64_t)floor(fabs(x) + 0.5);
                int64_t sc = x < 0 ? -c : c;
                t[k] = (c == 1) ? 1 : sc;
                col += (int)(c % 3) * mul;
                mul *= 3;
            }
            if (which == 2 + 2 * D) {  // task
                uint64_t tk = 0;
#pragma unroll
                for (int k = 0; k < D; ++k) tk |= ((uint64_t)(t[k] + (1 << 20)) & 0x1fffffull) << (21 * k);
                out = tk;
            } else {
                out = (uint64_t)col;
            }
        }
    }
    key[m] = out;
}

// run boundaries: abs keys (and colour/task when coloured) change
template <int D>
__global__ void k_run_flags(int64_t np, const uint32_t *__restrict__ P, const int32_t *__restrict__ pi,
                            const int32_t *__restrict__ pj, const double4 *__restrict__ XV,
                            double3 center, KSpec ks, int coloured, int64_t *flag) {
    int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= np) return;
    if (m == 0) { flag[0] = 1; return; }
    double cm[2][3];
    int64_t tk[2][3];
    for (int s = 0; s < 2; ++s) {
        const uint32_t p = P[m - s];
        const double4 a = XV[pi[p]], b = XV[pj[p]];
        const double ca[3] = {a.x, a.y, a.z}, cb[3] = {b.x, b.y, b.z};
        const double cen[3] = {center.x, center.y, center.z};
        for (int k = 0; k < D; ++k) {
            cm[s][k] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(ca[k], cb[k])), cen[k]);
            double x = cm[s][k] * ks.inv_h[k];
            int64_t c = (int64_t)floor(fabs(x) + 0.5);
            tk[s][k] = (c == 1) ? 1 : (x < 0 ? -c : c);
        }
    }
    bool brk = false;
    for (int k = 0; k < D; ++k) {
        brk |= fabs(cm[0][k]) != fabs(cm[1][k]);
        if (coloured) brk |= tk[0][k] != tk[1][k];
    }
    flag[m] = brk ? 1 : 0;
}

__global__ void k_run_starts(int64_t np, const int64_t *__restrict__ flag, const int64_t *__restrict__ scan,
                             int64_t *run_start) {
    int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= np) return;
    if (flag[m]) run_start[scan[m]] = m;
}

// split each run into particle-sharing components (neighbors.py:165);
// pass 0 counts groups per run, pass 1 writes the reordered pairs and
// group boundaries.
template <bool WRITE>
__global__ void k_split_runs(int64_t nruns, int64_t np, const int64_t *__restrict__ run_start,
                             const uint32_t *__restrict__ P, const int32_t *__restrict__ pi,
                             const int32_t *__restrict__ pj, int64_t *ngr,
                             const int64_t *__restrict__ goff, int32_t *opi, int32_t *opj,
                             int64_t *gptr, int *too_big) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    const int64_t lo = run_start[r], hi = (r + 1 < nruns) ? run_start[r + 1] : np;
    const int m = (int)(hi - lo);
    if (m == 1) {
        if (!WRITE) ngr[r] = 1;
        else {
            const uint32_t p = P[lo];
            opi[lo] = pi[p]; opj[lo] = pj[p];
            gptr[goff[r]] = lo;
        }
        return;
    }
    if (m > 64) { atomicExch(too_big, 1); if (!WRITE) ngr[r] = 1; return; }
    int32_t node[128];
    int par[128];
    int nn = 0;
    int ea[64], eb[64];
    for (int k = 0; k < m; ++k) {
        const uint32_t p = P[lo + k];
        int32_t e[2] = {pi[p], pj[p]};
        int idx[2];
        for (int s = 0; s < 2; ++s) {
            int f = -1;
            for (int t = 0; t < nn; ++t) if (node[t] == e[s]) { f = t; break; }
            if (f < 0) { node[nn] = e[s]; par[nn] = nn; f = nn++; }
            idx[s] = f;
        }
        ea[k] = idx[0]; eb[k] = idx[1];
        int ra = idx[0], rb = idx[1];
        while (par[ra] != ra) ra = par[ra];
        while (par[rb] != rb) rb = par[rb];
        if (ra != rb) { if (ra < rb) par[rb] = ra; else par[ra] = rb; }
    }
    int comp[64];
    int roots[64];
    int nc = 0;
    for (int k = 0; k < m; ++k) {
        int x = ea[k];
        while (par[x] != x) x = par[x];
        int f = -1;
        for (int t = 0; t < nc; ++t) if (roots[t] == x) { f = t; break; }
        if (f < 0) { roots[nc] = x; f = nc++; }
        comp[k] = f;
    }
    (void)eb;
    if (!WRITE) { ngr[r] = nc; return; }
    int64_t w = lo, g = goff[r];
    for (int c = 0; c < nc; ++c) {
        gptr[g++] = w;
        for (int k = 0; k < m; ++k)
            if (comp[k] == c) {
                const uint32_t p = P[lo + k];
                opi[w] = pi[p]; opj[w] = pj[p]; ++w;
            }
    }
}

__global__ void k_group_scratch(int64_t ng, const int64_t *__restrict__ gptr, int64_t *sz) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    int64_t m = gptr[g + 1] - gptr[g];
    int64_t nb = 2 * m;
    sz[g] = (m > 1) ? nb * nb + 4 * nb : 0;
}
__global__ void k_group_scratch_fix(int64_t ng, const int64_t *__restrict__ gptr, int64_t *off) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    if (gptr[g + 1] - gptr[g] <= 1) off[g] = -1;
}

// group-level task boundaries for the coloured schedule
template <int D>
__global__ void k_task_flags(int64_t ng, const int64_t *__restrict__ gptr, const int32_t *__restrict__ pi,
                             const int32_t *__restrict__ pj, const double4 *__restrict__ XV,
                             double3 center, KSpec ks, int64_t *flag, int32_t *colour) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= ng) return;
    int64_t tk[2][3];
    int col = 0;
    for (int s = 0; s < 2; ++s) {
        if (g - s < 0) break;
        const int64_t p = gptr[g - s];
        const double4 a = XV[pi[p]], b = XV[pj[p]];
        const double ca[3] = {a.x, a.y, a.z}, cb[3] = {b.x, b.y, b.z};
        const double cen[3] = {center.x, center.y, center.z};
        int mul = 1;
        for (int k = 0; k < D; ++k) {
            double cm = __dsub_rn(__dmul_rn(0.5, __dadd_rn(ca[k], cb[k])), cen[k]);
            double x = cm * ks.inv_h[k];
            int64_t c = (int64_t)floor(fabs(x) + 0.5);
            tk[s][k] = (c == 1) ? 1 : (x < 0 ? -c : c);
            if (s == 0) col += (int)(c % 3) * mul;
            mul *= 3;
        }
    }
    bool brk = (g == 0);
    if (g > 0) for (int k = 0; k < D; ++k) brk |= tk[0][k] != tk[1][k];
    flag[g] = brk ? 1 : 0;
    colour[g] = col;
}

// ------------------------------------------------------------ host build

inline KSpec make_kspec(int d, const double *h_axes) {
    static const double PI = 3.14159265358979323846;
    const double sigma[4] = {0.0, 3.0 / 4.0, 7.0 / (4.0 * PI), 21.0 / (16.0 * PI)};
    KSpec ks{};
    double prod = 1.0, hmin = h_axes[0];
    for (int k = 0; k < 3; ++k) { ks.inv_h[k] = 1.0; ks.h[k] = 1.0; ks.inv_h2[k] = 1.0; }
    for (int k = 0; k < d; ++k) {
        ks.h[k] = h_axes[k];
        ks.inv_h[k] = 1.0 / h_axes[k];
        ks.inv_h2[k] = ks.inv_h[k] * ks.inv_h[k];
        prod *= h_axes[k];
        hmin = std::min(hmin, h_axes[k]);
    }
    ks.pref = sigma[d] / prod;
    ks.pref5 = -5.0 * ks.pref;
    ks.h_min = hmin;
    return ks;
}

template <int D>
void build_schedule(NbhDev &nb, CubTemp &tmp, cudaStream_t s);

template <int D>
void build_nbh_impl(NbhDev &nb, const double *pos_h, const double *vol_h, cudaStream_t s) {
    const int64_t n = nb.n;
    CubTemp tmp;
    // bounding box of the scaled positions (host, O(n) scalar pass) and of
    // X for the pair-key centre (neighbors.py:102)
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, xlo[3] = {0, 0, 0}, xhi[3] = {0, 0, 0};
    for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < D; ++k) {
            double x = pos_h[i * D + k], u = x / nb.h_axes[k];
            if (i == 0 || u < lo[k]) lo[k] = u;
            if (i == 0 || u > hi[k]) hi[k] = u;
            if (i == 0 || x < xlo[k]) xlo[k] = x;
            if (i == 0 || x > xhi[k]) xhi[k] = x;
        }
    for (int k = 0; k < 3; ++k) nb.center[k] = 0.5 * (xlo[k] + xhi[k]);
    if (nb.has_grid) {
        // multi-rank: every rank bins on the GLOBAL cell grid, so a rank's
        // Morton order, blocks and pair lists are the global ones restricted
        for (int k = 0; k < D; ++k) { lo[k] = nb.grid_lo[k]; hi[k] = nb.grid_hi[k]; }
    }
    int dims[3] = {1, 1, 1};
    for (int k = 0; k < D; ++k) {
        double span = std::floor((hi[k] - lo[k]) * 0.5) + 1.0;
        if (span > (D == 3 ? 2097151.0 : 4294967295.0))
            throw Error(3, "particle cloud too extended for the cell grid");
        dims[k] = (int)span;
    }
    DBuf<double> pos(n * D), vol(n);
    pos.upload(pos_h, n * D, s);
    vol.upload(vol_h, n, s);
    DBuf<uint64_t> key(n), key2(n);
    DBuf<int64_t> val(n);
    nb.perm.alloc(n);
    nb.iperm.alloc(n);
    k_cell_keys<D><<<blocks_for(n), kThreads, 0, s>>>(n, pos.p, nb.ks, make_double3(lo[0], lo[1], lo[2]),
                                                      make_int3(dims[0], dims[1], dims[2]), key.p, val.p);
    MT_LAUNCH_CHECK();
    sort_pairs(tmp, key.p, key2.p, val.p, nb.perm.p, n, 64, s);
    nb.XV.alloc(n);
    DBuf<double4> U(n);
    k_gather_sorted<D><<<blocks_for(n), kThreads, 0, s>>>(n, nb.perm.p, pos.p, vol.p, nb.ks, nb.iperm.p,
                                                          nb.XV.p, U.p);
    MT_LAUNCH_CHECK();
    // occupied cells
    DBuf<int64_t> flag(n), scan(n), cell_of(n);
    k_cell_starts<<<blocks_for(n), kThreads, 0, s>>>(n, key2.p, flag.p);
    exclusive_scan(tmp, flag.p, scan.p, n, s);
    int64_t last_scan = 0, last_flag = 0;
    MT_CUDA(cudaMemcpyAsync(&last_scan, scan.p + n - 1, 8, cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaMemcpyAsync(&last_flag, flag.p + n - 1, 8, cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaStreamSynchronize(s));
    const int64_t ncell = last_scan + last_flag;
    DBuf<int64_t> cell_start(ncell);
    DBuf<uint64_t> cell_key(ncell);
    k_cell_index<<<blocks_for(n), kThreads, 0, s>>>(n, flag.p, scan.p, cell_of.p, cell_start.p, cell_key.p,
                                                    key2.p);
    DBuf<int32_t> cnb(ncell * 27);
    k_cell_neighbours<D><<<blocks_for(ncell), kThreads, 0, s>>>(ncell, cell_key.p,
                                                                make_int3(dims[0], dims[1], dims[2]), cnb.p);
    MT_LAUNCH_CHECK();
    // neighbour counts + duplicate detection
    DBuf<int64_t> count(n);
    DBuf<unsigned long long> dup(1);
    unsigned long long dup_h = ~0ull;
    dup.upload(&dup_h, 1, s);
    k_neigh<D, false><<<blocks_for(n), kThreads, 0, s>>>(n, U.p, cell_of.p, cell_start.p, ncell, cnb.p,
                                                         nb.perm.p, count.p, nullptr, nullptr, dup.p);
    MT_LAUNCH_CHECK();
    dup.download(&dup_h, 1, s);
    MT_CUDA(cudaStreamSynchronize(s));
    if (dup_h != ~0ull)
        throw Error(3, "duplicate particle positions (id " + std::to_string(dup_h) + ")", {(int64_t)dup_h});
    nb.indptr.alloc(n + 1);
    {
        DBuf<int64_t> cnt1(n + 1);
        MT_CUDA(cudaMemcpyAsync(cnt1.p, count.p, n * 8, cudaMemcpyDeviceToDevice, s));
        MT_CUDA(cudaMemsetAsync(cnt1.p + n, 0, 8, s));
        exclusive_scan(tmp, cnt1.p, nb.indptr.p, n + 1, s);
    }
    MT_CUDA(cudaMemcpyAsync(&nb.nnz, nb.indptr.p + n, 8, cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaStreamSynchronize(s));
    if (nb.nnz >= (int64_t)INT32_MAX * 2) throw Error(1, "neighbour table too large");
    nb.csr.alloc(std::max<int64_t>(nb.nnz, 1));
    k_neigh<D, true><<<blocks_for(n), kThreads, 0, s>>>(n, U.p, cell_of.p, cell_start.p, ncell, cnb.p,
                                                        nb.perm.p, nullptr, nb.indptr.p, nb.csr.p, nullptr);
    MT_LAUNCH_CHECK();
    // SELL-32 (only for the one-lane-per-particle gathers, MTSPH_GATHER_LANES=0)
    if (nb.want_sell) {
    nb.nslices = (n + 31) / 32;
    nb.slice_w.alloc(nb.nslices);
    nb.slice_ptr.alloc(nb.nslices + 1);
    {
        DBuf<int64_t> sz(nb.nslices + 1);
        MT_CUDA(cudaMemsetAsync(sz.p + nb.nslices, 0, 8, s));
        k_slice_width<<<blocks_for(nb.nslices), kThreads, 0, s>>>(n, nb.nslices, count.p, nb.slice_w.p, sz.p);
        exclusive_scan(tmp, sz.p, nb.slice_ptr.p, nb.nslices + 1, s);
    }
    MT_CUDA(cudaMemcpyAsync(&nb.sell_size, nb.slice_ptr.p + nb.nslices, 8, cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaStreamSynchronize(s));
    nb.nbr.alloc(std::max<int64_t>(nb.sell_size, 1));
    k_fill_sell<<<blocks_for(nb.nslices * 32), kThreads, 0, s>>>(n, nb.indptr.p, nb.csr.p, nb.slice_ptr.p,
                                                                 nb.slice_w.p, nb.nbr.p);
    MT_LAUNCH_CHECK();
    }
    // corrections
    nb.B.alloc(n * D * D);
    DBuf<uint8_t> sing(n);
    k_corrections<D><<<blocks_for(n), kThreads, 0, s>>>(n, nb.XV.p, nb.indptr.p, nb.csr.p, nb.ks, nb.B.p,
                                                        sing.p);
    MT_LAUNCH_CHECK();
    {
        std::vector<uint8_t> sh(n);
        std::vector<int64_t> perm_h(n);
        sing.download(sh.data(), n, s);
        nb.perm.download(perm_h.data(), n, s);
        MT_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> bad;
        for (int64_t k = 0; k < n; ++k)
            if (sh[k] && !(nb.ghost_orig && nb.ghost_orig[perm_h[k]])) bad.push_back(perm_h[k]);
        if (!bad.empty()) {
            std::sort(bad.begin(), bad.end());
            std::string ids;
            for (size_t k = 0; k < bad.size() && k < 10; ++k) ids += (k ? ", " : "") + std::to_string(bad[k]);
            throw Error(4, "singular kernel moment matrix at " + std::to_string(bad.size()) +
                               " particle(s), first ids: [" + ids + "]", bad);
        }
    }
    nb.cellkey = std::move(key2);
    if (nb.sweep == 1 || nb.sweep == 2) build_schedule<D>(nb, tmp, s);
    MT_CUDA(cudaStreamSynchronize(s));
}

template <int D>
void build_schedule(NbhDev &nb, CubTemp &tmp, cudaStream_t s) {
    const int64_t n = nb.n;
    // unique pairs, reference orientation
    DBuf<int64_t> pc(n + 1), poff(n + 1);
    MT_CUDA(cudaMemsetAsync(pc.p + n, 0, 8, s));
    k_pair_count<<<blocks_for(n), kThreads, 0, s>>>(n, nb.indptr.p, nb.csr.p, nb.perm.p, pc.p);
    exclusive_scan(tmp, pc.p, poff.p, n + 1, s);
    int64_t np = 0;
    MT_CUDA(cudaMemcpyAsync(&np, poff.p + n, 8, cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaStreamSynchronize(s));
    nb.npairs = np;
    if (np == 0) {
        nb.ngroups = 0;
        nb.gptr.alloc(1);
        int64_t z = 0;
        nb.gptr.upload(&z, 1, s);
        nb.level_ptr_h = {0};
        nb.colour_task_ptr = {0};
        nb.task_ptr.alloc(1);
        nb.task_ptr.upload(&z, 1, s);
        return;
    }
    if (np >= (int64_t)UINT32_MAX) throw Error(1, "too many pairs for the schedule");
    DBuf<int32_t> pi0(np), pj0(np);
    k_pair_fill<<<blocks_for(n), kThreads, 0, s>>>(n, nb.indptr.p, nb.csr.p, nb.perm.p, poff.p, pi0.p, pj0.p);
    MT_LAUNCH_CHECK();
    // stable radix sorts, least significant key first (np.lexsort order)
    DBuf<uint32_t> P(np), P2(np);
    k_iota<<<blocks_for(np), kThreads, 0, s>>>(np, P.p);
    DBuf<uint64_t> key(np), key2(np);
    const bool coloured = nb.sweep == 2;
    const int nkeys = 2 + 2 * D + (coloured ? 2 : 0);
    int id_bits = 1;
    while ((1ll << id_bits) <= n) ++id_bits;
    const double3 cen = make_double3(nb.center[0], nb.center[1], nb.center[2]);
    for (int which = 0; which < nkeys; ++which) {
        k_pair_key<D><<<blocks_for(np), kThreads, 0, s>>>(np, P.p, pi0.p, pj0.p, nb.perm.p, nb.XV.p, cen, nb.ks,
                                                          which, key.p);
        MT_LAUNCH_CHECK();
        int bits = (which < 2) ? id_bits : (which == 2 + 2 * D + 1 ? 8 : 64);
        sort_pairs(tmp, key.p, key2.p, P.p, P2.p, np, bits, s);
        std::swap(P.p, P2.p);
    }
    // runs and groups
    DBuf<int64_t> flag(np), scan(np);
    k_run_flags<D><<<blocks_for(np), kThreads, 0, s>>>(np, P.p, pi0.p, pj0.p, nb.XV.p, cen, nb.ks,
                                                       coloured ? 1 : 0, flag.p);
    exclusive_scan(tmp, flag.p, scan.p, np, s);
    int64_t ls = 0, lf = 0;
    MT_CUDA(cudaMemcpyAsync(&ls, scan.p + np - 1, 8, cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaMemcpyAsync(&lf, flag.p + np - 1, 8, cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaStreamSynchronize(s));
    const int64_t nruns = ls + lf;
    DBuf<int64_t> run_start(nruns), ngr(nruns + 1), goff(nruns + 1);
    k_run_starts<<<blocks_for(np), kThreads, 0, s>>>(np, flag.p, scan.p, run_start.p);
    DBuf<int> too_big(1);
    too_big.zero(s);
    MT_CUDA(cudaMemsetAsync(ngr.p + nruns, 0, 8, s));
    k_split_runs<false><<<blocks_for(nruns, 128), 128, 0, s>>>(nruns, np, run_start.p, P.p, pi0.p, pj0.p, ngr.p,
                                                          nullptr, nullptr, nullptr, nullptr, too_big.p);
    MT_LAUNCH_CHECK();
    exclusive_scan(tmp, ngr.p, goff.p, nruns + 1, s);
    int tb = 0;
    too_big.download(&tb, 1, s);
    MT_CUDA(cudaMemcpyAsync(&nb.ngroups, goff.p + nruns, 8, cudaMemcpyDeviceToHost, s));
    MT_CUDA(cudaStreamSynchronize(s));
    if (tb) throw Error(3, "degenerate lattice: more than 64 interacting pairs share a damping group key");
    nb.pi.alloc(np);
    nb.pj.alloc(np);
    nb.gptr.alloc(nb.ngroups + 1);
    MT_CUDA(cudaMemcpyAsync(nb.gptr.p + nb.ngroups, &np, 8, cudaMemcpyHostToDevice, s));
    k_split_runs<true><<<blocks_for(nruns, 128), 128, 0, s>>>(nruns, np, run_start.p, P.p, pi0.p, pj0.p, nullptr,
                                                         goff.p, nb.pi.p, nb.pj.p, nb.gptr.p, too_big.p);
    MT_LAUNCH_CHECK();
    const int64_t ng = nb.ngroups;
    // scratch for simultaneous group solves
    {
        DBuf<int64_t> sz(ng + 1);
        nb.gscr.alloc(ng + 1);
        MT_CUDA(cudaMemsetAsync(sz.p + ng, 0, 8, s));
        k_group_scratch<<<blocks_for(ng), kThreads, 0, s>>>(ng, nb.gptr.p, sz.p);
        exclusive_scan(tmp, sz.p, nb.gscr.p, ng + 1, s);
        MT_CUDA(cudaMemcpyAsync(&nb.scratch_doubles, nb.gscr.p + ng, 8, cudaMemcpyDeviceToHost, s));
        k_group_scratch_fix<<<blocks_for(ng), kThreads, 0, s>>>(ng, nb.gptr.p, nb.gscr.p);
        MT_CUDA(cudaStreamSynchronize(s));
        nb.scratch.alloc(std::max<int64_t>(nb.scratch_doubles, 1));
    }
    if (!coloured) {
        // level schedule of the serial order: level(g) = 1 + max over its
        // particles of the level of the previous group touching them
        std::vector<int32_t> hpi(np), hpj(np);
        std::vector<int64_t> hg(ng + 1);
        nb.pi.download(hpi.data(), np, s);
        nb.pj.download(hpj.data(), np, s);
        nb.gptr.download(hg.data(), ng + 1, s);
        MT_CUDA(cudaStreamSynchronize(s));
        std::vector<int32_t> last(n, 0), lev(ng);
        int32_t maxl = 0;
        for (int64_t g = 0; g < ng; ++g) {
            int32_t L = 0;
            for (int64_t k = hg[g]; k < hg[g + 1]; ++k) L = std::max(L, std::max(last[hpi[k]], last[hpj[k]]));
            ++L;
            for (int64_t k = hg[g]; k < hg[g + 1]; ++k) last[hpi[k]] = last[hpj[k]] = L;
            lev[g] = L;
            maxl = std::max(maxl, L);
        }
        nb.nlevels = maxl;
        nb.level_ptr_h.assign(maxl + 1, 0);
        for (int64_t g = 0; g < ng; ++g) nb.level_ptr_h[lev[g]]++;
        for (int32_t L = 1; L <= maxl; ++L) nb.level_ptr_h[L] += nb.level_ptr_h[L - 1];
        std::vector<int64_t> fillp(nb.level_ptr_h.begin(), nb.level_ptr_h.end() - 1), lg(ng);
        for (int64_t g = 0; g < ng; ++g) lg[fillp[lev[g] - 1]++] = g;
        nb.level_groups.upload(lg.data(), ng, s);
    } else {
        DBuf<int64_t> tf(ng), ts(ng);
        DBuf<int32_t> col(ng);
        k_task_flags<D><<<blocks_for(ng), kThreads, 0, s>>>(ng, nb.gptr.p, nb.pi.p, nb.pj.p, nb.XV.p, cen, nb.ks,
                                                            tf.p, col.p);
        MT_LAUNCH_CHECK();
        std::vector<int64_t> htf(ng);
        std::vector<int32_t> hcol(ng);
        tf.download(htf.data(), ng, s);
        col.download(hcol.data(), ng, s);
        MT_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> tptr;
        std::vector<int32_t> tcol;
        for (int64_t g = 0; g < ng; ++g)
            if (htf[g]) { tptr.push_back(g); tcol.push_back(hcol[g]); }
        nb.ntasks = (int64_t)tptr.size();
        tptr.push_back(ng);
        // tasks are sorted by colour (most significant key)
        int ncol = 1;
        for (int k = 0; k < D; ++k) ncol *= 3;
        nb.colour_task_ptr.assign(ncol + 1, 0);
        for (int64_t t = 0; t < nb.ntasks; ++t) nb.colour_task_ptr[tcol[t] + 1]++;
        for (int c = 0; c < ncol; ++c) nb.colour_task_ptr[c + 1] += nb.colour_task_ptr[c];
        nb.task_ptr.upload(tptr.data(), tptr.size(), s);
        MT_CUDA(cudaStreamSynchronize(s));
    }
}

inline void build_nbh(NbhDev &nb, int64_t n, int d, const double *pos, const double *vol,
                      const double *h_axes, int sweep, cudaStream_t s) {
    if (d != 2 && d != 3) throw Error(1, "device neighbourhoods support d = 2 or 3");
    if (n <= 0) throw Error(1, "empty particle set");
    if (n >= (int64_t)INT32_MAX) throw Error(1, "too many particles for int32 neighbour ids");
    for (int64_t i = 0; i < n; ++i) {
        if (!(vol[i] > 0.0)) throw Error(3, "volumes must be positive, one per particle");
        for (int k = 0; k < d; ++k)
            if (!std::isfinite(pos[i * d + k])) throw Error(3, "non-finite reference positions");
    }
    for (int k = 0; k < d; ++k)
        if (!(h_axes[k] > 0.0)) throw Error(1, "smoothing length must be positive");
    nb.n = n;
    nb.d = d;
    nb.sweep = sweep;
    for (int k = 0; k < 3; ++k) nb.h_axes[k] = k < d ? h_axes[k] : 1.0;
    nb.ks = make_kspec(d, h_axes);
    if (d == 2) build_nbh_impl<2>(nb, pos, vol, s);
    else build_nbh_impl<3>(nb, pos, vol, s);
}

}  // namespace mtsph
