// window.cuh -- 3D neighbour gathers from shared-memory cell windows.
//
// The two per-step neighbour gathers (solids.py:118 deformation_rate ->
// _accel.py:16 velocity_gradient_gather, and solids.py:170
// stress_divergence_acceleration -> _accel.py:34 pair_tensor_divergence)
// read, for every particle, ~78 neighbour records.  From global memory
// (gather_csr.cuh) each warp load touches ~12 different 128 B lines and the
// L1 data stage moves ~48 B per wavefront: the kernels are bound by the
// LSU data pipe at 15-22 % of HBM.  Here the records come from shared
// memory instead, where a conflict-free LDS.128 moves 128 B per wavefront.
//
// Cells have the kernel support as edge, so every neighbour of a particle
// lies in the 3 x 3 x 3 cells around its own.  A CTA walks a pencil of
// target cells along x (a task: cells (x0..x1-1, y, z)).  The window of
// target cell X is three slabs, X-1, X, X+1, each the 3 x 3 cells
// (X, y-1..y+1, z-1..z+1); moving to X+1 only loads one more slab.  Slabs
// live in a ring of five slots (three in use, two loading: prefetch
// distance two target cells), staged with 16 B cp.async copies (coalesced:
// a cell is a contiguous particle range in the Morton order); the target
// cell's row pointers and neighbour entries ride in the same groups.
//
// A neighbour entry is addressed by a precomputed 16-bit slab-local id,
// wl = (dx + 1) << 14 | offset in slab X + dx (setup, k_win_index), so the
// inner loop is: wl -> ring slot -> 2 or 3 swizzled records.  Records are
// 32 B planes; 16 B half h of record r sits at chunk 2r + (h ^ bit2(r)), so
// the eight lanes of a quarter warp reading eight consecutive records hit
// eight different 16 B bank groups.
//
// A target cell's ~18 particles share the CTA: G = threads / count lanes
// per particle walk its CSR row with stride G, the per-lane partial sums go
// to shared memory, are summed in lane order (deterministic) and the
// epilogue is the CSR kernels' (F update; a = ... with the static G term).
// Sum order differs from the CSR gathers by rounding only.
//
// Measured (B200, 10M-particle bench bar, profiles/tuning_r02/window_*):
// parity holds (100-step trajectory at 1e-10), but the gathers are SLOWER
// than the CSR ones -- stress 9.9 ms and accel 9.7 ms per step against 5.6
// and 5.9 -- so this path is opt-in (MTSPH_GATHER_WINDOW=1).  ncu (2M
// slice): the inner loop costs what the CSR loop costs (~80 thread
// instructions per neighbour visit), but a target cell gives each thread
// only ~6 visits between barriers, and the per-cell work around them
// (staging issue, row copies, lane split, reductions, stores: ~550 warp
// instructions per warp and cell) is as large again; 119 registers and
// 94-112 KB of shared memory leave 16 warps per SM, and 40 % of the
// shared-memory wavefronts are bank conflicts (a quarter warp straddles two
// particles' rows).  First version (prefetch distance one, per-thread
// 9-way chunk selection, epilogues in the kernel): 13 / 14 ms.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "solid.cuh"

namespace mtsph {

struct WinSched {
    bool on = false;
    int cap = 0;           // records per slab slot (multiple of 8)
    int wcap = 0;          // u16 neighbour entries per target-cell slot (multiple of 8)
    int icap = 0;          // int64 row pointers per target-cell slot (even)
    int threads = 256;     // threads per CTA
    int seg = 16;          // target cells per task
    int64_t ntasks = 0;
    int gdim[3] = {0, 0, 0};
    int max_cell = 0;
    DBuf<int4> tasks;      // (y, z, x0, x1), bbox cell coordinates
    DBuf<int4> cell;       // dense bbox grid (first particle, count, row entries, -), x fastest
    DBuf<uint16_t> wl;     // per CSR entry
};

struct WinArgs {
    const int4 *tasks;
    const int4 *cell;
    const uint16_t *wl;
    const int64_t *indptr;
    int gx, gy, gz;
    int cap, wcap, icap;
};

constexpr int kWinSlots = 5;  // slab ring: three in use, two loading
constexpr int kWinTSlots = 3; // target-cell ring (rows + entries): one in use, two loading

// shared-memory chunk (16 B) of half h of slab record r
__device__ __forceinline__ int wswz(int r, int h) { return 2 * r + (h ^ ((r >> 2) & 1)); }

__device__ __forceinline__ double2 lds2(const double4 *base, int r, int h) {
    return *reinterpret_cast<const double2 *>(reinterpret_cast<const char *>(base) + 16 * wswz(r, h));
}

__device__ __forceinline__ int4 win_cell(const WinArgs &W, int x, int y, int z) {
    if (x < 0 || x >= W.gx || y < 0 || y >= W.gy || z < 0 || z >= W.gz) return make_int4(0, 0, 0, 0);
    return __ldg(W.cell + ((int64_t)z * W.gy + y) * W.gx + x);
}

__device__ __forceinline__ void cp16(void *dst, const void *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait2() { asm volatile("cp.async.wait_group 2;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// Shared-memory layout of one CTA (window kernels)
struct WinSmem {
    double4 *ring;      // [kWinSlots][NP][cap] swizzled records
    uint16_t *wls;      // [kWinTSlots][wcap]
    int64_t *ips;       // [kWinTSlots][icap]
    int *meta;          // [kWinTSlots][8]: count, entry shift, row shift, first particle, G, per
    int *cofs;          // [kWinSlots]: offset of the slab's centre cell
    double *part;       // [threads][K]
};
template <int NP, int K> __device__ __forceinline__ WinSmem win_smem_map(void *base, const WinArgs &W) {
    WinSmem m;
    char *p = reinterpret_cast<char *>(base);
    m.ring = reinterpret_cast<double4 *>(p);
    p += (size_t)kWinSlots * NP * W.cap * sizeof(double4);
    m.ips = reinterpret_cast<int64_t *>(p);
    p += (size_t)kWinTSlots * W.icap * sizeof(int64_t);
    m.part = reinterpret_cast<double *>(p);
    p += (size_t)blockDim.x * K * sizeof(double);
    m.wls = reinterpret_cast<uint16_t *>(p);
    p += (size_t)kWinTSlots * W.wcap * sizeof(uint16_t);
    m.meta = reinterpret_cast<int *>(p);
    m.cofs = m.meta + kWinTSlots * 8;
    return m;
}
inline size_t win_smem_bytes(int cap, int wcap, int icap, int threads, int np, int k) {
    return (size_t)kWinSlots * np * cap * 32 + (size_t)kWinTSlots * icap * 8 + (size_t)threads * k * 8 +
           (size_t)kWinTSlots * wcap * 2 + (size_t)(kWinTSlots * 8 + kWinSlots) * 4;
}

// cp.async the NP record planes of slab x (cells (x, y+dy, z+dz), (dz, dy)
// row-major) into its ring slot, and (tgt) the rows and neighbour entries
// of target cell (x-1, y, z) into its target slot.  Warp w copies cells w,
// w + nwarps, ...: lanes 0..8 read the nine cell entries, a shuffle scan
// gives the offsets, then the warp streams its cells' records (consecutive
// lanes: consecutive 16 B of one cell).  The caller commits the group.
template <int NP>
__device__ __forceinline__ void win_issue(const WinArgs &W, const double4 *const *planes, const WinSmem &m,
                                          int x, int y, int z, bool slab, bool tgt) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (slab) {
        const int slot = ((x % kWinSlots) + kWinSlots) % kWinSlots;
        int4 c = make_int4(0, 0, 0, 0);
        if (lane < 9) c = win_cell(W, x, y + lane % 3 - 1, z + lane / 3 - 1);
        int pre = c.y;  // inclusive scan over lanes 0..8
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, pre, o);
            if (lane >= o) pre += t;
        }
        pre -= c.y;  // exclusive
        if (threadIdx.x == 4) m.cofs[slot] = pre;
        for (int j = warp; j < 9; j += nw) {
            const int st = __shfl_sync(0xffffffffu, c.x, j), cnt = __shfl_sync(0xffffffffu, c.y, j),
                      r0 = __shfl_sync(0xffffffffu, pre, j);
            for (int q = lane; q < 2 * cnt; q += 32) {
                const int r = r0 + (q >> 1), h = q & 1;
#pragma unroll
                for (int p = 0; p < NP; ++p)
                    cp16(reinterpret_cast<char *>(m.ring + (size_t)(slot * NP + p) * W.cap) + 16 * wswz(r, h),
                         reinterpret_cast<const char *>(planes[p] + st + (q >> 1)) + 16 * h);
            }
        }
    }
    if (tgt) {
        // target cell (x-1, y, z): its particles' row pointers and entries,
        // copied in aligned 16 B chunks (meta holds the shifts and the lane
        // split: G lanes per particle, per particles per round)
        const int4 tc = win_cell(W, x - 1, y, z);
        const int ts = ((x - 1) % kWinTSlots + kWinTSlots) % kWinTSlots;
        const int64_t f0 = tc.x & ~1ll;                       // int64 rows: 2 per chunk
        const int nic = (int)(((int64_t)tc.x + tc.y + 2 - f0) >> 1);
        int64_t e0 = 0;
        if (tc.y > 0) e0 = __ldg(W.indptr + tc.x);
        const int64_t eb = e0 & ~7ll;                          // u16 entries: 8 per chunk
        const int nwc = (int)((e0 + tc.z - eb + 7) >> 3);
        if (threadIdx.x == 0) {
            const int T = (int)blockDim.x;
            const int G = tc.y >= T ? 1 : T / max(tc.y, 1);
            m.meta[ts * 8 + 0] = tc.y;
            m.meta[ts * 8 + 1] = (int)(e0 - eb);
            m.meta[ts * 8 + 2] = (int)(tc.x - f0);
            m.meta[ts * 8 + 3] = tc.x;
            m.meta[ts * 8 + 4] = G;
            m.meta[ts * 8 + 5] = T / G;
        }
        for (int c = threadIdx.x; c < nic + nwc; c += blockDim.x) {
            if (c < nic) cp16(m.ips + (size_t)ts * W.icap + 2 * c, W.indptr + f0 + 2 * c);
            else cp16(m.wls + (size_t)ts * W.wcap + 8 * (c - nic), W.wl + eb + 8 * (c - nic));
        }
    }
}

// The pencil walk shared by both gathers.  Body(X, ts, p, sub, G, acc)
// gathers local particle p of target cell X over lanes sub of G into
// acc[K]; Out(i, k, v) stores component k of particle i's sum.
template <int NP, int K, class Body, class Out>
__device__ __forceinline__ void win_walk(const WinArgs &W, const double4 *const *planes, const WinSmem &m,
                                         const uint8_t *flags, Body body, Out out) {
    const int4 tk = W.tasks[blockIdx.x];
    const int y = tk.x, z = tk.y, x0 = tk.z, x1 = tk.w;
    const int T = (int)blockDim.x;
    // group A: slabs x0-1 .. x0+1 and target x0; group B: slab x0+2, target x0+1
    win_issue<NP>(W, planes, m, x0 - 1, y, z, true, false);
    win_issue<NP>(W, planes, m, x0, y, z, true, false);
    win_issue<NP>(W, planes, m, x0 + 1, y, z, true, true);
    cp_commit();
    win_issue<NP>(W, planes, m, x0 + 2, y, z, x0 + 2 <= x1, x0 + 1 < x1);
    cp_commit();
    for (int X = x0; X < x1; ++X) {
        __syncthreads();  // target X-1 done: slab slot of X-2, target slot of X-1 and the partials are free
        win_issue<NP>(W, planes, m, X + 3, y, z, X + 3 <= x1, X + 2 < x1);
        cp_commit();
        cp_wait2();
        __syncthreads();  // slabs X-1..X+1 and target X landed (every thread's copies)
        const int ts = X % kWinTSlots;
        const int nt = m.meta[ts * 8 + 0];
        if (nt == 0) continue;
        const int first = m.meta[ts * 8 + 3], G = m.meta[ts * 8 + 4], per = m.meta[ts * 8 + 5];
        // lane split: exact for threadIdx < 2^12 (a float quotient of small integers)
        const int p0 = (int)((float)threadIdx.x / (float)G), sub = (int)threadIdx.x - p0 * G;
        for (int base = 0; base < nt; base += per) {
            const int npr = min(per, nt - base);
            double acc[K];
#pragma unroll
            for (int k = 0; k < K; ++k) acc[k] = 0.0;
            if (p0 < npr) body(X, ts, base + p0, sub, G, acc);
#pragma unroll
            for (int k = 0; k < K; ++k) m.part[threadIdx.x * K + k] = acc[k];
            __syncthreads();
            // lane-order sums, in place into the particle's first lane slot
            for (int q = threadIdx.x; q < npr * K; q += T) {
                const int pp = q / K, kk = q - pp * K;
                const double *pq = m.part + pp * G * K + kk;
                double s = 0.0;
                for (int j = 0; j < G; ++j) s += pq[j * K];
                m.part[pp * G * K + kk] = s;
            }
            __syncthreads();
            for (int q = threadIdx.x; q < npr * K; q += T) {  // coalesced SoA stores
                const int kk = (int)((float)q / (float)npr), pp = q - kk * npr;
                const int64_t i = (int64_t)first + base + pp;
                if (!(flags[i] & FL_GHOST)) out(i, kk, m.part[pp * G * K + kk]);
            }
            if (base + per < nt) __syncthreads();
        }
    }
    cp_wait0();
}

// Row of local particle p of target slot ts: [lo, hi) into m.wls
__device__ __forceinline__ void win_row(const WinArgs &W, const WinSmem &m, int ts, int p, int &lo, int &hi) {
    const int64_t *ip = m.ips + (size_t)ts * W.icap + m.meta[ts * 8 + 2];
    const int64_t r0 = ip[0];
    lo = (int)(ip[p] - r0) + m.meta[ts * 8 + 1];
    hi = (int)(ip[p + 1] - r0) + m.meta[ts * 8 + 1];
}

// ring slots of slabs X-1, X, X+1 (plane 0 of each)
template <int NP>
__device__ __forceinline__ void win_bases(const WinSmem &m, const WinArgs &W, int X, const double4 *(&b)[3]) {
#pragma unroll
    for (int d = 0; d < 3; ++d) b[d] = m.ring + (size_t)(((X + d - 1 + kWinSlots) % kWinSlots) * NP) * W.cap;
}

// sum_b V_b (v_b - v_a) (x) gradW  ->  Lacc (F is updated in k_solid_rmap)
__global__ void __launch_bounds__(256, 2) k_win_stress(SolidArgs A, WinArgs W) {
    extern __shared__ double4 wsm[];
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const int64_t n = A.n;
    const WinSmem m = win_smem_map<2, 9>(wsm, W);
    const double4 *planes[2] = {A.XV, reinterpret_cast<const double4 *>(A.V)};
    double *Lacc = const_cast<double *>(A.Lacc);
    auto body = [&](int X, int ts, int p, int sub, int G, double *acc) {
        const double4 *bs[3];
        win_bases<2>(m, W, X, bs);
        const int ra = m.cofs[X % kWinSlots] + p;  // in the centre slab
        const double2 xa01 = lds2(bs[1], ra, 0), xa2v = lds2(bs[1], ra, 1);
        const double2 va01 = lds2(bs[1] + W.cap, ra, 0), va2p = lds2(bs[1] + W.cap, ra, 1);
        int lo, hi;
        win_row(W, m, ts, p, lo, hi);
        const uint16_t *wr = m.wls + (size_t)ts * W.wcap;
        for (int k = lo + sub; k < hi; k += G) {
            const unsigned w = wr[k];
            const unsigned dx = w >> 14;
            const int r = (int)(w & 0x3fffu);
            const double4 *b0 = dx == 0 ? bs[0] : (dx == 1 ? bs[1] : bs[2]), *b1 = b0 + W.cap;
            const double2 x01 = lds2(b0, r, 0), x2v = lds2(b0, r, 1);
            const double2 v01 = lds2(b1, r, 0), v2p = lds2(b1, r, 1);
            const double rel[3] = {x01.x - xa01.x, x01.y - xa01.y, x2v.x - xa2v.x};
            double g[3];
            grad_w<3>(rel, A.ks, g);
            const double volb = x2v.y;
            const double dv[3] = {volb * (v01.x - va01.x), volb * (v01.y - va01.y), volb * (v2p.x - va2p.x)};
#pragma unroll
            for (int r2 = 0; r2 < 3; ++r2)
#pragma unroll
                for (int cc = 0; cc < 3; ++cc) acc[r2 * 3 + cc] += dv[r2] * g[cc];
        }
    };
    auto out = [&](int64_t i, int k, double v) { Lacc[(int64_t)k * n + i] = v; };
    win_walk<2, 9>(W, planes, m, A.flags, body, out);
}

// sum_b T~_b gradW -> a (k_solid_kick_part adds T_a G_a / V_a, divides by
// rho0, kicks and reduces, as k_solid_accel_csr's epilogue)
__global__ void __launch_bounds__(256, 2) k_win_accel(SolidArgs A, WinArgs W) {
    extern __shared__ double4 wsm[];
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const int64_t n = A.n;
    const WinSmem m = win_smem_map<3, 3>(wsm, W);
    const double4 *tp = reinterpret_cast<const double4 *>(A.T);
    const double4 *planes[3] = {tp, tp + n, tp + 2 * n};
    auto body = [&](int X, int ts, int p, int sub, int G, double *acc) {
        const double4 *bs[3];
        win_bases<3>(m, W, X, bs);
        const double4 *a2 = bs[1] + 2 * W.cap;
        const int ra = m.cofs[X % kWinSlots] + p;
        const double2 xa01 = lds2(a2, ra, 0), xa2t = lds2(a2, ra, 1);
        int lo, hi;
        win_row(W, m, ts, p, lo, hi);
        const uint16_t *wr = m.wls + (size_t)ts * W.wcap;
        for (int k = lo + sub; k < hi; k += G) {
            const unsigned w = wr[k];
            const unsigned dx = w >> 14;
            const int r = (int)(w & 0x3fffu);
            const double4 *b0 = dx == 0 ? bs[0] : (dx == 1 ? bs[1] : bs[2]), *b1 = b0 + W.cap, *b2 = b1 + W.cap;
            const double2 t01 = lds2(b0, r, 0), t23 = lds2(b0, r, 1);
            const double2 t45 = lds2(b1, r, 0), t67 = lds2(b1, r, 1);
            const double2 x01 = lds2(b2, r, 0), x2t = lds2(b2, r, 1);
            const double rel[3] = {x01.x - xa01.x, x01.y - xa01.y, x2t.x - xa2t.x};
            double g[3];
            grad_w<3>(rel, A.ks, g);
            acc[0] = fma(t01.x, g[0], acc[0]);
            acc[0] = fma(t01.y, g[1], acc[0]);
            acc[0] = fma(t23.x, g[2], acc[0]);
            acc[1] = fma(t23.y, g[0], acc[1]);
            acc[1] = fma(t45.x, g[1], acc[1]);
            acc[1] = fma(t45.y, g[2], acc[1]);
            acc[2] = fma(t67.x, g[0], acc[2]);
            acc[2] = fma(t67.y, g[1], acc[2]);
            acc[2] = fma(x2t.y, g[2], acc[2]);
        }
    };
    auto out = [&](int64_t i, int k, double v) { A.a[(int64_t)k * n + i] = v; };
    win_walk<3, 3>(W, planes, m, A.flags, body, out);
}

// a = (sum + T_a G_a / V_a) / rho0, v += dt/2 a for movable particles, E_k
// and |a|max block partials (k_solid_accel_csr's epilogue, after a window
// gather)
template <int D>
__global__ void __launch_bounds__(256) k_solid_kick_part(SolidArgs A) {
    using V_t = typename VT<D>::T;
    __shared__ double sh[32];
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int64_t n = A.n;
    double ek = 0.0, a2m = 0.0;
    if (i < n && !(A.flags[i] & FL_GHOST)) {
        const uint8_t f = A.flags[i];
        double Ta[D * D], xd[3], acc[D];
        dload<D>(A.T, n, A.XV, i, Ta, xd);
        const double rho0 = A.rho0[i], vola = volof<D>(ldg4(A.XV + i));
#pragma unroll
        for (int k = 0; k < D; ++k) {
            double ta = 0.0;
#pragma unroll
            for (int cc = 0; cc < D; ++cc) ta += Ta[k * D + cc] * A.G[(int64_t)cc * n + i];
            acc[k] = (A.a[(int64_t)k * n + i] + ta / vola) / rho0;
            A.a[(int64_t)k * n + i] = acc[k];
        }
        if (f & FL_MOVABLE) {
            const double dt = c->dt;
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
            V_t w;
            vset(w, v);
            V[i] = w;
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

// ------------------------------------------------------------- setup

__device__ __forceinline__ uint32_t compact3(uint64_t v) {  // every 3rd bit -> 21 bits
    v &= 0x1249249249249249ull;
    v = (v ^ (v >> 2)) & 0x10c30c30c30c30c3ull;
    v = (v ^ (v >> 4)) & 0x100f00f00f00f00full;
    v = (v ^ (v >> 8)) & 0x1f0000ff0000ffull;
    v = (v ^ (v >> 16)) & 0x1f00000000ffffull;
    v = (v ^ (v >> 32)) & 0x1fffffull;
    return (uint32_t)v;
}

// slab-local id of every CSR entry; err bit 1: a neighbour outside the 27
// cells, bit 2: a slab offset >= 2^14
__global__ void k_win_index(int64_t n, const uint64_t *__restrict__ cellkey, const int64_t *__restrict__ indptr,
                            const int32_t *__restrict__ csr, WinArgs W, int3 org, uint16_t *wl, int *err) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t ka = cellkey[i];
    const int cx = (int)compact3(ka) - org.x, cy = (int)compact3(ka >> 1) - org.y,
              cz = (int)compact3(ka >> 2) - org.z;
    int off[27];
    for (int dx = 0; dx < 3; ++dx) {
        int pre = 0;
        for (int j = 0; j < 9; ++j) {
            off[dx * 9 + j] = pre;
            pre += win_cell(W, cx + dx - 1, cy + j % 3 - 1, cz + j / 3 - 1).y;
        }
    }
    int e = 0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) {
        const int32_t b = csr[k];
        const uint64_t kb = cellkey[b];
        const int dx = (int)compact3(kb) - org.x - cx, dy = (int)compact3(kb >> 1) - org.y - cy,
                  dz = (int)compact3(kb >> 2) - org.z - cz;
        if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) { e |= 1; continue; }
        const int4 cb = win_cell(W, cx + dx, cy + dy, cz + dz);
        const int o = off[(dx + 1) * 9 + (dz + 1) * 3 + (dy + 1)] + (b - cb.x);
        if (o >= (1 << 14)) { e |= 2; continue; }
        wl[k] = (uint16_t)((dx + 1) << 14 | o);
    }
    if (e) atomicOr(err, e);
}

inline size_t win_smem(const WinSched &w, int np, int k) {
    return win_smem_bytes(w.cap, w.wcap, w.icap, w.threads, np, k);
}

inline WinArgs win_args(const WinSched &w, const NbhDev &nb) {
    return WinArgs{w.tasks.p, w.cell.p,    w.wl.p, nb.indptr.p, w.gdim[0], w.gdim[1], w.gdim[2],
                   w.cap,     w.wcap,      w.icap};
}

// Build the window schedule of a 3D neighbourhood; leaves w.on = false
// (CSR gathers) when a slab or the grid is too large.  MTSPH_GATHER_WINDOW=1
// enables it, MTSPH_WIN_SEG sets the target cells per task.
inline void build_window(const NbhDev &nb, WinSched &w, cudaStream_t s) {
    w = WinSched();
    if (nb.d != 3 || nb.n == 0) return;
    // opt-in (measured slower than the CSR gathers at 10M, see the header)
    if (const char *e = std::getenv("MTSPH_GATHER_WINDOW"); !e || e[0] != '1') return;
    if (const char *e = std::getenv("MTSPH_WIN_SEG")) w.seg = std::max(1, std::atoi(e));
    const int64_t n = nb.n;
    std::vector<uint64_t> key(n);
    std::vector<int64_t> ip(n + 1);
    nb.cellkey.download(key.data(), n, s);
    nb.indptr.download(ip.data(), n + 1, s);
    MT_CUDA(cudaStreamSynchronize(s));
    auto dec = [](uint64_t k, int a) {
        uint32_t v = 0;
        for (int b = 0; b < 21; ++b) v |= (uint32_t)((k >> (3 * b + a)) & 1ull) << b;
        return (int)v;
    };
    // occupied cells
    struct Cell { int c[3]; int start, cnt; };
    std::vector<Cell> cells;
    for (int64_t i = 0; i < n; ++i) {
        if (i == 0 || key[i] != key[i - 1]) {
            if (i > (int64_t)INT32_MAX) return;
            cells.push_back({{dec(key[i], 0), dec(key[i], 1), dec(key[i], 2)}, (int)i, 0});
        }
        ++cells.back().cnt;
    }
    int lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
    for (const Cell &c : cells)
        for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], c.c[a]); hi[a] = std::max(hi[a], c.c[a]); }
    for (int a = 0; a < 3; ++a) w.gdim[a] = hi[a] - lo[a] + 1;
    const int64_t gcells = (int64_t)w.gdim[0] * w.gdim[1] * w.gdim[2];
    if (gcells > (int64_t)1 << 28) return;
    std::vector<int4> grid((size_t)gcells, make_int4(0, 0, 0, 0));
    int64_t max_ent = 0;
    auto lin = [&](int x, int y, int z) { return ((int64_t)z * w.gdim[1] + y) * w.gdim[0] + x; };
    for (const Cell &c : cells) {
        const int64_t ne = ip[c.start + c.cnt] - ip[c.start];
        if (ne > (int64_t)1 << 20) return;
        max_ent = std::max(max_ent, ne);
        grid[lin(c.c[0] - lo[0], c.c[1] - lo[1], c.c[2] - lo[2])] = make_int4(c.start, c.cnt, (int)ne, 0);
        w.max_cell = std::max(w.max_cell, c.cnt);
    }
    auto cnt = [&](int x, int y, int z) {
        if (x < 0 || y < 0 || z < 0 || x >= w.gdim[0] || y >= w.gdim[1] || z >= w.gdim[2]) return 0;
        return grid[lin(x, y, z)].y;
    };
    // largest slab (3 x 3 cells) -> ring slot capacity
    int cap = 0;
    for (int z = 0; z < w.gdim[2]; ++z)
        for (int y = 0; y < w.gdim[1]; ++y)
            for (int x = 0; x < w.gdim[0]; ++x) {
                int t = 0;
                for (int j = 0; j < 9; ++j) t += cnt(x, y + j % 3 - 1, z + j / 3 - 1);
                cap = std::max(cap, t);
            }
    w.cap = (cap + 7) & ~7;
    if (w.cap == 0 || w.cap > (1 << 14)) return;
    // target-cell slots: aligned 16 B copies add up to 7 entries / 1 row on
    // each side
    w.wcap = (int)((max_ent + 16 + 7) & ~7);
    w.icap = (w.max_cell + 4 + 1) & ~1;
    // smem: the accel window (3 planes) is the larger one; two CTAs per SM
    // are wanted, one must fit
    int dev = 0, optin = 0;
    MT_CUDA(cudaGetDevice(&dev));
    MT_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (win_smem(w, 3, 3) > (size_t)optin) return;
    // tasks: pencil segments holding at least one occupied target cell
    std::vector<int4> tasks;
    for (int z = 0; z < w.gdim[2]; ++z)
        for (int y = 0; y < w.gdim[1]; ++y) {
            int xa = -1, xb = -1;
            for (int x = 0; x < w.gdim[0]; ++x)
                if (cnt(x, y, z)) { if (xa < 0) xa = x; xb = x; }
            if (xa < 0) continue;
            for (int x0 = xa; x0 <= xb; x0 += w.seg) {
                const int x1 = std::min(xb + 1, x0 + w.seg);
                bool any = false;
                for (int x = x0; x < x1 && !any; ++x) any = cnt(x, y, z) > 0;
                if (any) tasks.push_back(make_int4(y, z, x0, x1));
            }
        }
    w.ntasks = (int64_t)tasks.size();
    w.tasks.upload(tasks.data(), tasks.size(), s);
    w.cell.upload(grid.data(), grid.size(), s);
    w.wl.alloc((size_t)std::max<int64_t>(nb.nnz, 1) + 16);  // + the aligned copies' overrun
    w.wl.zero(s);
    DBuf<int> err(1);
    err.zero(s);
    WinArgs W = win_args(w, nb);
    k_win_index<<<blocks_for(n), 256, 0, s>>>(n, nb.cellkey.p, nb.indptr.p, nb.csr.p, W,
                                               make_int3(lo[0], lo[1], lo[2]), w.wl.p, err.p);
    MT_LAUNCH_CHECK();
    int herr = 0;
    err.download(&herr, 1, s);
    MT_CUDA(cudaStreamSynchronize(s));
    if (herr) {
        std::fprintf(stderr, "[mtsph] window gathers disabled (index check %d)\n", herr);
        w = WinSched();
        return;
    }
    allow_max_dynamic_smem((const void *)k_win_stress);
    allow_max_dynamic_smem((const void *)k_win_accel);
    w.on = true;
    if (const char *e = std::getenv("MTSPH_VERBOSE"); e && e[0] == '1')
        std::fprintf(stderr,
                     "[mtsph] window gathers: grid %d x %d x %d cells, %lld tasks of <= %d cells, slab cap %d, "
                     "max cell %d, entry slot %d, smem stress %zu B accel %zu B\n",
                     w.gdim[0], w.gdim[1], w.gdim[2], (long long)w.ntasks, w.seg, w.cap, w.max_cell, w.wcap,
                     win_smem(w, 2, 9), win_smem(w, 3, 3));
}


}  // namespace mtsph
