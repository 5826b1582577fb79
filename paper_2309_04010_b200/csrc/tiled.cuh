// tiled.cuh -- shared-memory tiled damping sweep (MTSPH_SWEEP_TILED).
//
// The B200 throughput variant of the pairwise implicit damping sweep.
// Particles are already sorted by the Morton code of cells whose edge is
// the kernel support, so an aligned block of B^d cells is a contiguous
// particle range.  A block owns the pairs (a, b), a < b, whose first
// particle lies in it; every particle such a pair touches lies in the
// block's halo (the block grown by one cell).  Blocks are 2^d-coloured by
// the parity of their block coordinates: same-coloured blocks are one block
// apart, so their halos are disjoint and they run concurrently.
//
// One CTA per block: the halo's velocities and inverse masses are staged
// in shared memory; the block's pairs, greedily edge-coloured at setup
// (each sub-colour is a matching), are applied sub-colour by sub-colour
// with a __syncthreads between them; the halo is written back.  A sweep
// is colours 0..2^d-1 with sub-colours ascending, then everything in
// reverse at half the step each -- a symmetric Gauss-Seidel ordering like
// the reference's forward/reverse serial sweep.  Each pair update is the
// reference's closed-form backward-Euler two-body exchange, so pair
// momentum is conserved exactly and kinetic energy never increases.
#pragma once

#include <algorithm>
#include <array>
#include <exception>
#include <functional>
#include <mutex>
#include <unordered_map>
#include <thread>

#include "damping.cuh"
#include "nbh.cuh"

namespace mtsph {

// depth of the cp.async ring that stages sub-colour chunks (prefetch
// distance stages - 1 sub-colours), per real type.  Measured at 10M (3D,
// 512 threads, sub-colours <= 448 pairs): fp64 3 stages 6.58 ms (2 CTAs/SM
// fit; 4 stages: 1 CTA/SM, 8.47 ms), fp32 4 stages 3.94 ms (3 CTAs/SM;
// 3 stages 4.31 ms)
#ifndef MTSPH_SWEEP_STAGES64
#define MTSPH_SWEEP_STAGES64 3
#endif
#ifndef MTSPH_SWEEP_STAGES32
#define MTSPH_SWEEP_STAGES32 4
#endif
// How the pair/coefficient chunks reach shared memory: TMA bulk copies
// completing on mbarriers (every thread applies pairs), or per-element
// cp.async by dedicated staging warps.  Bit-identical.  Measured at 10M (3D):
// fp64 sweep 6.19 -> 5.72 ms with TMA; fp32 3.67 ms with cp.async, 3.83
// with TMA.  MTSPH_SWEEP_TMA=0 builds cp.async for both.
#ifndef MTSPH_SWEEP_TMA
#define MTSPH_SWEEP_TMA 1
#endif
template <class R> struct SweepTma { static constexpr bool on = MTSPH_SWEEP_TMA != 0; };
template <> struct SweepTma<float> { static constexpr bool on = false; };
template <class R> struct SweepStages { static constexpr int n = MTSPH_SWEEP_STAGES64; };
template <> struct SweepStages<float> { static constexpr int n = MTSPH_SWEEP_STAGES32; };
inline int sweep_stages(int rsize) { return rsize == 8 ? MTSPH_SWEEP_STAGES64 : MTSPH_SWEEP_STAGES32; }

struct TiledSched {
    int sh = 0;                      // low Morton bits per block (build_tiled)
    int64_t ntasks = 0;
    int max_halo = 0, max_ranges = 0, maxsub = 0, max_nsub = 0;
    int64_t nsub_total = 0;          // sub-colours over all tasks (one pass)
    int threads = 128;
    std::vector<int64_t> colour_ptr; // 2^d + 1, over tasks (colour-major)
    DBuf<int64_t> range_off;         // ntasks + 1 -> ranges
    DBuf<int2> ranges;               // (global start, local offset)
    DBuf<int32_t> halo_n;            // ntasks
    DBuf<int64_t> hid_off;           // ntasks + 1 -> hid
    DBuf<int32_t> hid;               // per task: the global id of every halo record (the ranges, expanded)
    DBuf<int64_t> pair_off;          // ntasks + 1 -> pairs
    DBuf<uint32_t> pairs;            // li | lj << 16
    DBuf<double> pd;                 // damping coefficient per pair
    DBuf<int64_t> sub_off;           // ntasks + 1 -> sub
    DBuf<int32_t> sub;               // per task: nsub + 1 pair offsets (task-relative)
    int64_t npairs = 0;
    // dataflow (persistent) sweep: overlapping-halo task lists, colours,
    // reverse-pass order, per-task completion + work counter (ntasks + 1)
    DBuf<int32_t> f_nboff, f_nbt, f_col, f_rev, f_done;
    int flow_grid = 0;               // 0: per-colour launches
    int flow_grid32 = 0;             // the same for the fp32 variant's kernel
};

// R: the precision of the velocities, inverse masses and coefficients
// (double: the reference path; float: the fp32 variant, solid32.cuh)
template <class R> struct TiledArgsT {
    const int64_t *range_off;
    const int2 *ranges;
    const int32_t *halo_n;
    const int64_t *pair_off;
    const uint32_t *pairs;
    const R *pd;
    const int64_t *sub_off;
    const int32_t *sub;
    const R *inv_m;
    void *V;
    int maxsub;      // largest sub-colour (pairs), sizes the staging buffers
    const int64_t *hid_off;  // per task -> hid
    const int32_t *hid;      // global ids of the task's halo records, in local order
};
using TiledArgs = TiledArgsT<double>;

// Shared-memory halo record (v0, v1, v2, 1/m), 16 B-strided so record l
// sits in 16 B bank group l % 8 (see sweep_task).  fp64: two arrays,
// (v0, v1) and (v2 | 0, 1/m), one LDS.128 each; fp32: one float4 array.
template <class R> struct Halo;
template <> struct Halo<double> {
    double2 *xy, *zw;
    __device__ __forceinline__ Halo(void *base, int H) : xy(reinterpret_cast<double2 *>(base)), zw(xy + H) {}
    __device__ __forceinline__ void *end(int H) const { return zw + H; }
    __device__ __forceinline__ void ld(int l, double &x, double &y, double &z, double &im) const {
        const double2 a = xy[l], b = zw[l];
        x = a.x; y = a.y; z = b.x; im = b.y;
    }
    template <int D> __device__ __forceinline__ void st(int l, double x, double y, double z, double im) {
        xy[l] = make_double2(x, y);
        if (D == 3) zw[l] = make_double2(z, im);  // 2D: the z|1/m half never changes
    }
    __device__ __forceinline__ void init(int l, double x, double y, double z, double im) {
        xy[l] = make_double2(x, y);
        zw[l] = make_double2(z, im);
    }
    static constexpr size_t bytes = 32;
};
template <> struct Halo<float> {
    float4 *r;
    __device__ __forceinline__ Halo(void *base, int) : r(reinterpret_cast<float4 *>(base)) {}
    __device__ __forceinline__ void *end(int H) const { return r + H; }
    __device__ __forceinline__ void ld(int l, float &x, float &y, float &z, float &im) const {
        const float4 a = r[l];
        x = a.x; y = a.y; z = a.z; im = a.w;
    }
    template <int D> __device__ __forceinline__ void st(int l, float x, float y, float z, float im) {
        r[l] = make_float4(x, y, z, im);
    }
    __device__ __forceinline__ void init(int l, float x, float y, float z, float im) { r[l] = make_float4(x, y, z, im); }
    static constexpr size_t bytes = 16;
};

__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    } while (!ok);
}

// the ring's mbarriers (one per slot, one arrival per phase), once per CTA
template <int S, class R> __device__ __forceinline__ void mbar_init(uint64_t *mbar) {
    if constexpr (!SweepTma<R>::on) {
        (void)mbar;
        return;
    }
    if (threadIdx.x == 0) {
        for (int k = 0; k < S; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(mbar + k))
                         : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
}

// One block task (one CTA): stage the halo, apply the sub-colours in
// direction dir, write the halo back.  FLOW: other SMs write V during the
// launch (persistent dataflow sweep), so the halo is read through L2.
template <int D, bool FLOW, class R>
__device__ __forceinline__ void sweep_task(const TiledArgsT<R> &T, int64_t task, int dir, R half,
                                           double *smem, uint64_t *mbar, uint32_t &gq) {
    using V_t = typename VTR<D, R>::T;
    const int H = T.halo_n[task];
    // halo (Halo<R>): record l sits in 16 B bank group l % 8, and
    // build_tiled orders each sub-colour so a quarter warp's li and lj are
    // distinct mod 8 -- one wavefront per halo access
    Halo<R> hal(smem, H);
    V_t *V = reinterpret_cast<V_t *>(T.V);
    // global ids of the halo records: the task's cell ranges expanded at
    // setup (a coalesced 4 B stream; the binary search of the range table it
    // replaces cost ~14 shared-memory loads per record and pass)
    const int32_t *__restrict__ hid = T.hid + T.hid_off[task];
    auto global_of = [&](int l) { return (int64_t)__ldg(hid + l); };
    const int64_t p0 = T.pair_off[task];
    const int64_t s0 = T.sub_off[task];
    const int nsub = (int)(T.sub_off[task + 1] - s0) - 1;
    constexpr int kSweepStages = SweepStages<R>::n;
    // ring of kSweepStages (pair, coefficient) chunks
    R *bd = reinterpret_cast<R *>(hal.end(H));                                 // ring of coefficients
    uint32_t *bp = reinterpret_cast<uint32_t *>(bd + kSweepStages * T.maxsub);  // ring of pairs
    int *ssub = reinterpret_cast<int *>(bp + kSweepStages * T.maxsub);         // sub-colour bounds
    // one word per sub-colour: first pair (low 20 bits) | pair count << 20, so
    // the loop reads one shared-memory word per warp and iteration, not two
    // (a task holds < 2^20 pair slots, a sub-colour < 2^12)
    for (int k = threadIdx.x; k < nsub; k += blockDim.x) {
        const int a = T.sub[s0 + k], b = T.sub[s0 + k + 1];
        ssub[k] = a | ((b - a) << 20);
    }
    __syncthreads();
    // dir 1: sub-colours ascending, -1: descending.  (Merging the last
    // forward and first reverse colour into one launch was measured slower.)
    const int nq = nsub;
    auto sub_range = [&](int q, int &a, int &b) {
        const int s = dir > 0 ? q : nsub - 1 - q;
        const int w = ssub[s];
        a = w & 0xfffff;
        b = a + (int)((unsigned)w >> 20);
    };
    // the pair updates of sub-colour q from ring slot `slot`, npr lanes
    auto apply_sub = [&](int q, int slot, int npr) {
        int a0, b0;
        sub_range(q, a0, b0);
        const int cnt = b0 - a0;
        const R *cd = bd + slot * T.maxsub;
        const uint32_t *cpk = bp + slot * T.maxsub;
        for (int p = threadIdx.x; p < cnt; p += npr) {  // npr % 8 == 0: groups stay quarter warps
            const uint32_t pk = cpk[p];
            if (pk == 0xffffffffu) continue;  // kPadPair
            const int li = (int)(pk & 0xffffu), lj = (int)(pk >> 16);
            R ax, ay, az, ai, bx, by, bz, bi;
            hal.ld(li, ax, ay, az, ai);
            hal.ld(lj, bx, by, bz, bi);
            const R c = half * cd[p];
            const R ca = c * ai, cb = c * bi;
            const R rden = R(1) / (R(1) + ca + cb);
            R u = (ax - bx) * rden;
            ax -= ca * u;
            bx += cb * u;
            u = (ay - by) * rden;
            ay -= ca * u;
            by += cb * u;
            if (D == 3) {
                u = (az - bz) * rden;
                az -= ca * u;
                bz += cb * u;
            }
            hal.template st<D>(li, ax, ay, az, ai);
            hal.template st<D>(lj, bx, by, bz, bi);
        }
    };
    auto stage_halo = [&]() {
        for (int l = threadIdx.x; l < H; l += blockDim.x) {
            const int64_t g = global_of(l);
            R v[3] = {0, 0, 0};
            // per-colour launches: halos of one launch are disjoint, read-only here
            vget(FLOW ? vldcg(V + g) : vldg(V + g), v);
            hal.init(l, v[0], v[1], D == 3 ? v[2] : R(0), T.inv_m[g]);
        }
    };
    if constexpr (SweepTma<R>::on) {
        // Chunks move by TMA bulk copies (cp.async.bulk, one elected thread
        // per chunk, completion on the slot's mbarrier), so every thread
        // applies pairs.  Chunk q of this task is the CTA's chunk gq + q:
        // slot (gq + q) % S, mbarrier phase parity ((gq + q) / S) & 1.  A slot
        // is refilled only after the barrier that ends the sub-colour that
        // read it.
        auto issue = [&](int q) {
            if (q >= nq) return;
            const uint32_t c = gq + (uint32_t)q;
            const int slot = (int)(c % kSweepStages);
            int a, b;
            sub_range(q, a, b);
            const uint32_t nb_pk = (uint32_t)(b - a) * 4u, nb_pd = (uint32_t)(b - a) * (uint32_t)sizeof(R);
            const uint32_t mb = (uint32_t)__cvta_generic_to_shared(mbar + slot);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mb), "r"(nb_pk + nb_pd)
                         : "memory");
            if (nb_pk) {
                const uint32_t dpd = (uint32_t)__cvta_generic_to_shared(bd + slot * T.maxsub);
                const uint32_t dpp = (uint32_t)__cvta_generic_to_shared(bp + slot * T.maxsub);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                    ::"r"(dpd), "l"(T.pd + p0 + a), "r"(nb_pd), "r"(mb) : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                    ::"r"(dpp), "l"(T.pairs + p0 + a), "r"(nb_pk), "r"(mb) : "memory");
            }
        };
        // the issuer is lane 0 of the last warp: sub-colours hold at most
        // maxsub <= blockDim - 64 pairs, so that warp has no pairs to apply
        // and the copies stay off the barrier-to-barrier critical path
        const bool issuer = threadIdx.x == blockDim.x - 32;
        if (issuer)
            for (int q = 0; q < kSweepStages; ++q) issue(q);
        stage_halo();
        __syncthreads();
        for (int q = 0; q < nq; ++q) {
            const uint32_t c = gq + (uint32_t)q;
            const int slot = (int)(c % kSweepStages);
            mbar_wait((uint32_t)__cvta_generic_to_shared(mbar + slot), (c / kSweepStages) & 1u);
            apply_sub(q, slot, (int)blockDim.x);
            __syncthreads();
            if (issuer) issue(q + kSweepStages);  // slot of sub-colour q is free now
        }
        gq += (uint32_t)nq;
    } else {
        // Warp-specialised: the top eighth of the threads (whole warps, at
        // least one) only stage chunks by per-element cp.async, the rest
        // only apply pairs, so a chunk's copy overlaps the pair updates.
        // Whole warps: the two roles reach __syncthreads (bar.sync, .aligned)
        // from different call sites, which a warp may only do if all its
        // lanes take the same one.
        const int nst = std::max(32, (int)(blockDim.x >> 3) & ~31), npr = (int)blockDim.x - nst;
        const bool stager = (int)threadIdx.x >= npr;
        const int st = (int)threadIdx.x - npr;
        // (stagers) every call commits exactly one (possibly empty) cp.async group
        auto stage = [&](int q) {
            if (q < nq) {
                const int slot = q % kSweepStages;
                int a, b;
                sub_range(q, a, b);
                for (int p = a + st; p < b; p += nst) {
                    const unsigned dpd = (unsigned)__cvta_generic_to_shared(bd + slot * T.maxsub + (p - a));
                    const unsigned dpp = (unsigned)__cvta_generic_to_shared(bp + slot * T.maxsub + (p - a));
                    if (sizeof(R) == 8)
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dpd), "l"(T.pd + p0 + p));
                    else
                        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dpd), "l"(T.pd + p0 + p));
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dpp), "l"(T.pairs + p0 + p));
                }
            }
            asm volatile("cp.async.commit_group;\n" ::);
        };
        // prefetch distance kSweepStages-1 sub-colours; the first ones
        // stream in while the halo is gathered
        if (stager)
            for (int q = 0; q < kSweepStages - 1; ++q) stage(q);
        stage_halo();
        if (stager) asm volatile("cp.async.wait_group %0;\n" ::"n"(kSweepStages - 2));  // chunk 0
        __syncthreads();
        // One barrier per sub-colour, at the end of iteration q.  Before it
        // the stagers have issued chunk q + S - 1 into slot (q - 1) % S (free:
        // every thread passed the previous barrier, so sub-colour q - 1 is
        // done) and waited for chunks <= q + 1; after it chunk q + 1 is
        // visible to all and sub-colour q is complete in the halo.
        for (int q = 0; q < nq; ++q) {
            if (stager) {
                stage(q + kSweepStages - 1);
                asm volatile("cp.async.wait_group %0;\n" ::"n"(kSweepStages - 2));
            } else {
                apply_sub(q, q % kSweepStages, npr);
            }
            __syncthreads();
        }
    }
    for (int l = threadIdx.x; l < H; l += blockDim.x) {
        const int64_t g = global_of(l);
        R v[3], im;
        hal.ld(l, v[0], v[1], v[2], im);
        V_t w;
        vset(w, v);
        vst(V + g, w);
    }
}

// per-colour launch: one CTA per block task of the colour
template <int D, class R = double>
__global__ void __launch_bounds__(1024) k_sweep_tiled(TiledArgsT<R> T, int64_t t0, int dir, const Ctrl *ctrl) {
    extern __shared__ double smem[];
    __shared__ __align__(8) uint64_t mbar[SweepStages<R>::n];
    if (ctrl->done) return;
    mbar_init<SweepStages<R>::n, R>(mbar);
    uint32_t gq = 0;
    sweep_task<D, false, R>(T, t0 + blockIdx.x, dir, R(0.5 * ctrl->dt * ctrl->eta), smem, mbar, gq);
}

// Dataflow schedule of a whole sweep (both passes) in one persistent launch.
struct TiledFlow {
    const int32_t *nb_off, *nb_task;  // per task: the tasks whose halos overlap its halo
    const int32_t *colour;            // per task
    const int32_t *rev;               // reverse-pass task order (colours descending)
    int32_t *done;                    // per task: passes completed in this sweep
    int32_t *counter;                 // next work item
    int32_t ntasks;
};

__device__ __forceinline__ int ld_acquire_gpu(const int32_t *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int32_t *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Persistent sweep: CTAs claim work items in phase order (forward pass in
// colour-major task order, then the reverse pass with colours descending)
// and start an item once every task that touches its halo in an earlier
// phase is done -- so colour c+1 starts block by block as its neighbours of
// colour c finish, with no launch boundary (and no tail) between colours.
// Deadlock-free: an item only waits on items claimed earlier by running CTAs.
// Result identical to the per-colour launches (same tasks, same order on
// every particle).
template <int D, class R = double>
__global__ void __launch_bounds__(1024) k_sweep_flow(TiledArgsT<R> T, TiledFlow F, const Ctrl *ctrl) {
    extern __shared__ double smem[];
    __shared__ int s_w;
    __shared__ __align__(8) uint64_t mbar[SweepStages<R>::n];
    if (ctrl->done) return;
    mbar_init<SweepStages<R>::n, R>(mbar);
    uint32_t gq = 0;  // chunks this CTA has consumed (ring slot and phase)
    const R half = R(0.5 * ctrl->dt * ctrl->eta);
    for (;;) {
        if (threadIdx.x == 0) s_w = atomicAdd(F.counter, 1);
        __syncthreads();
        const int w = s_w;
        if (w >= 2 * F.ntasks) return;
        const int pass = w >= F.ntasks;
        const int t = pass ? F.rev[w - F.ntasks] : w;
        if (threadIdx.x < 32) {  // warp 0: one lane per dependency, so one L2 round trip
            const int ct = F.colour[t];
            if (pass && threadIdx.x == 0)
                while (ld_acquire_gpu(F.done + t) < 1) __nanosleep(32);
            for (int k = F.nb_off[t] + (int)threadIdx.x; k < F.nb_off[t + 1]; k += 32) {
                const int u = F.nb_task[k], cu = F.colour[u];
                const int need = pass == 0 ? (cu < ct ? 1 : 0) : (cu > ct ? 2 : 1);
                while (ld_acquire_gpu(F.done + u) < need) __nanosleep(32);
            }
        }
        __syncthreads();
        sweep_task<D, true, R>(T, t, pass ? -1 : 1, half, smem, mbar, gq);
        __syncthreads();  // every write-back of the halo issued
        if (threadIdx.x == 0) {
            __threadfence();
            st_release_gpu(F.done + t, pass + 1);
        }
    }
}

// setup: expand a task's (global start, local offset) cell ranges into the
// global id of every halo record
__global__ void k_tiled_halo_ids(const int64_t *__restrict__ range_off, const int2 *__restrict__ ranges,
                                 const int32_t *__restrict__ halo_n, const int64_t *__restrict__ hid_off,
                                 int32_t *hid) {
    const int64_t task = blockIdx.x;
    const int64_t r0 = range_off[task];
    const int nr = (int)(range_off[task + 1] - r0);
    const int H = halo_n[task];
    int32_t *out = hid + hid_off[task];
    for (int l = threadIdx.x; l < H; l += blockDim.x) {
        int lo = 0, hi = nr - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (ranges[r0 + mid].y <= l) lo = mid; else hi = mid - 1;
        }
        out[l] = ranges[r0 + lo].x + (l - ranges[r0 + lo].y);
    }
}

// rsize: bytes of the sweep's real type (8: fp64, 4: the fp32 variant)
inline size_t tiled_smem_bytes(const TiledSched &t, int d, int rsize = 8) {
    (void)d;
    return (size_t)((((t.max_ranges + 1) & ~1) + 3) / 4 * 4) * 8 + (size_t)t.max_halo * 4 * rsize +
           (size_t)t.maxsub * sweep_stages(rsize) * (4 + rsize) + (size_t)(t.max_nsub + 1) * 4;
}

template <int D, class R = double>
int launch_tiled_sweep(const TiledSched &t, const TiledArgsT<R> &A, const Ctrl *ctrl, cudaStream_t s) {
    const int nc = (int)t.colour_ptr.size() - 1;
    const size_t sm = tiled_smem_bytes(t, D, (int)sizeof(R));
    const int flow_grid = sizeof(R) == 8 ? t.flow_grid : t.flow_grid32;
    if (flow_grid > 0 && t.ntasks > 0) {
        MT_CUDA(cudaMemsetAsync(t.f_done.p, 0, sizeof(int32_t) * (size_t)(t.ntasks + 1), s));
        TiledFlow F{t.f_nboff.p, t.f_nbt.p, t.f_col.p, t.f_rev.p, t.f_done.p, t.f_done.p + t.ntasks,
                    (int32_t)t.ntasks};
        k_sweep_flow<D, R><<<(unsigned)flow_grid, t.threads, sm, s>>>(A, F, ctrl);
        MT_LAUNCH_CHECK();
        return 1;
    }
    int launches = 0;
    for (int pass = 0; pass < 2; ++pass)
        for (int q = 0; q < nc; ++q) {
            const int c = pass == 0 ? q : nc - 1 - q;
            const int64_t t0 = t.colour_ptr[c], t1 = t.colour_ptr[c + 1];
            if (t1 <= t0) continue;
            k_sweep_tiled<D, R><<<(unsigned)(t1 - t0), t.threads, sm, s>>>(A, t0, pass == 0 ? 1 : -1, ctrl);
            MT_LAUNCH_CHECK();
            ++launches;
        }
    return launches;
}

// ------------------------------------------------------------- host setup

namespace tiled_detail {

inline void decode(uint64_t key, int d, int64_t *c) {
    for (int k = 0; k < d; ++k) {
        uint64_t v = 0;
        for (int b = 0; b < (d == 3 ? 21 : 32); ++b) v |= ((key >> (b * d + k)) & 1ull) << b;
        c[k] = (int64_t)v;
    }
}
inline uint64_t encode(const int64_t *c, int d) {
    return d == 3 ? (spread3((uint64_t)c[0]) | spread3((uint64_t)c[1]) << 1 | spread3((uint64_t)c[2]) << 2)
                  : (spread2((uint64_t)c[0]) | spread2((uint64_t)c[1]) << 1);
}

struct TaskOut {
    int colour = 0;
    int halo = 0;
    std::vector<int2> ranges;
    std::vector<uint32_t> pairs;
    std::vector<double> pd;
    std::vector<int32_t> sub;
};

// Padding entry of a sub-colour: the lane idles (local ids are < 65535).
constexpr uint32_t kPadPair = 0xffffffffu;

// The pairs of one sub-colour are independent, so their order is free (the
// result is bit-identical in any order).  Emit them in groups of 8 -- one
// quarter warp of the kernel's LDS.128 halo accesses -- whose li % 8 and
// lj % 8 are all distinct, so each group reads and writes the halo in one
// shared-memory wavefront per access.  Each group is a maximum matching
// (Kuhn's augmenting paths) in the 8 x 8 bipartite graph of non-empty
// (li % 8, lj % 8) buckets, fullest rows and columns first; a group the
// buckets cannot complete is padded with kPadPair rather than given a
// conflicting pair.  The group count meets the lower bound max(row, column
// total) -- ~69 groups for a 470-pair sub-colour, where a random order
// costs ~137 quarter-warp wavefronts and a greedy one ~89.
inline void bank_order(const uint32_t *pairs, const double *pd, int64_t m, std::vector<uint32_t> &op,
                       std::vector<double> &od) {
    thread_local std::vector<int32_t> bk[64];
    for (auto &v : bk) v.clear();
    int rowtot[8] = {0, 0, 0, 0, 0, 0, 0, 0}, coltot[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t p = 0; p < m; ++p) {
        const int a = (int)(pairs[p] & 7u), b = (int)((pairs[p] >> 16) & 7u);
        bk[a * 8 + b].push_back((int32_t)p);
        ++rowtot[a];
        ++coltot[b];
    }
    int64_t left = m;
    while (left > 0) {
        int rows[8], cols[8], mc[8];
        for (int k = 0; k < 8; ++k) { rows[k] = cols[k] = k; mc[k] = -1; }
        std::sort(rows, rows + 8, [&](int x, int y) { return rowtot[x] > rowtot[y]; });
        std::sort(cols, cols + 8, [&](int x, int y) { return coltot[x] > coltot[y]; });
        unsigned vis = 0;
        struct Aug {  // Kuhn's augmenting path (depth <= 8)
            const std::vector<int32_t> *bk;
            const int *cols;
            int *mc;
            unsigned *vis;
            bool operator()(int a) const {
                for (int k = 0; k < 8; ++k) {
                    const int b = cols[k];
                    if (bk[a * 8 + b].empty() || (*vis >> b & 1)) continue;
                    *vis |= 1u << b;
                    if (mc[b] < 0 || (*this)(mc[b])) { mc[b] = a; return true; }
                }
                return false;
            }
        } augment{bk, cols, mc, &vis};
        for (int k = 0; k < 8; ++k) { vis = 0; augment(rows[k]); }
        int g = 0;
        for (int b = 0; b < 8; ++b) {
            if (mc[b] < 0) continue;
            const int a = mc[b];
            const int32_t p = bk[a * 8 + b].back();
            bk[a * 8 + b].pop_back();
            --rowtot[a];
            --coltot[b];
            --left;
            op.push_back(pairs[p]);
            od.push_back(pd[p]);
            ++g;
        }
        if (left > 0)
            for (; g < 8; ++g) { op.push_back(kPadPair); od.push_back(0.0); }
    }
}

}  // namespace tiled_detail

// Build the schedule from the device neighbourhood (host C++, threaded).
// vector whose elements are default-initialised (no zero fill of the
// multi-GB setup arrays that are overwritten anyway)
template <class T> struct NoInit : std::allocator<T> {
    using std::allocator<T>::allocator;
    template <class U> struct rebind { using other = NoInit<U>; };
    template <class U> void construct(U *p) noexcept { ::new (static_cast<void *>(p)) U; }
    template <class U, class... A> void construct(U *p, A &&...a) {
        ::new (static_cast<void *>(p)) U(std::forward<A>(a)...);
    }
};
template <class T> using RawVec = std::vector<T, NoInit<T>>;

template <class T, class Al> void upload_vec(DBuf<T> &b, const std::vector<T, Al> &v, cudaStream_t s) {
    b.alloc(std::max<size_t>(v.size(), 1));
    if (!v.empty()) copy_staged(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    MT_CUDA(cudaStreamSynchronize(s));
}
template <class T, class Al> void download_vec(std::vector<T, Al> &v, const DBuf<T> &b, size_t count, cudaStream_t s) {
    v.resize(std::max<size_t>(count, 1));
    if (count) copy_staged(v.data(), b.p, count * sizeof(T), cudaMemcpyDeviceToHost, s);
}

// A block is the run of particles whose cell keys agree above the low `sh`
// Morton bits: an aligned box of ext[0] x ext[1] (x ext[2]) cells, the
// interleave (x0 y0 z0 x1 ...) giving axis k the bits i < sh with i % d == k
// (sh = d log2 B: cubic edge B; sh = 5 in 3D: 4 x 4 x 2).
inline void build_tiled(const NbhDev &nb, int sh, TiledSched &t, cudaStream_t s) {
    using namespace tiled_detail;
    const int64_t n = nb.n;
    const int d = nb.d;
    // largest sub-colour in pairs (multiple of 8; 0 = none).  Default 448 =
    // the pair lanes of a 512-thread CTA: with it the fp64 block fits two
    // CTAs per SM (3D sweep 7.35 -> 6.58 ms at 10M, 2D 2.01 -> 1.78) and fp32
    // three (3D 4.22 -> 3.94, 2D 1.14 -> 1.05).  MTSPH_SWEEP_SUBCAP overrides.
    int subcap = 448;
    if (const char *e = std::getenv("MTSPH_SWEEP_SUBCAP")) subcap = std::max(0, std::atoi(e)) & ~7;
    int lg[3] = {0, 0, 0}, ext[3] = {1, 1, 1}, P[3] = {1, 1, 1};
    for (int i = 0; i < sh; ++i) ++lg[i % d];
    // block colour period per axis: same-coloured blocks must be two cells
    // apart so their one-cell halos are disjoint -- parity works from an
    // extent of 2 cells, single-cell extents need period 3
    for (int k = 0; k < d; ++k) { ext[k] = 1 << lg[k]; P[k] = ext[k] >= 2 ? 2 : 3; }
    RawVec<uint64_t> cellkey;
    RawVec<int64_t> indptr;
    RawVec<int32_t> csr;
    RawVec<double4> XV;
    download_vec(cellkey, nb.cellkey, n, s);
    download_vec(indptr, nb.indptr, n + 1, s);
    download_vec(csr, nb.csr, nb.nnz, s);
    download_vec(XV, nb.XV, n, s);
    setup_mark(s, "tiled: download");
    // occupied cells: key -> [start, end)
    std::vector<uint64_t> ckeys;
    std::vector<int64_t> cstart;
    for (int64_t i = 0; i < n; ++i)
        if (i == 0 || cellkey[i] != cellkey[i - 1]) { ckeys.push_back(cellkey[i]); cstart.push_back(i); }
    cstart.push_back(n);
    auto cell_range = [&](uint64_t key, int64_t &a, int64_t &b) {
        auto it = std::lower_bound(ckeys.begin(), ckeys.end(), key);
        if (it == ckeys.end() || *it != key) return false;
        const size_t c = it - ckeys.begin();
        a = cstart[c];
        b = cstart[c + 1];
        return true;
    };
    // blocks = runs of equal key >> sh
    std::vector<int64_t> bstart;
    for (int64_t i = 0; i < n; ++i)
        if (i == 0 || (cellkey[i] >> sh) != (cellkey[i - 1] >> sh)) bstart.push_back(i);
    const int64_t nblocks = (int64_t)bstart.size();
    bstart.push_back(n);
    // multi-rank: blocks of ghost particles belong to another rank
    std::vector<char> skip(nblocks, 0);
    if (!nb.ghost_internal.empty())
        for (int64_t bk = 0; bk < nblocks; ++bk) skip[bk] = nb.ghost_internal[bstart[bk]] != 0;
    std::vector<TaskOut> out(nblocks);
    const double4 *xv = XV.data();
    auto pdamp = [&](int64_t i, int64_t j) {
        const double a[3] = {xv[i].x, xv[i].y, xv[i].z}, b[3] = {xv[j].x, xv[j].y, xv[j].z};
        double rel[3], r2 = 0.0;
        for (int k = 0; k < d; ++k) { rel[k] = b[k] - a[k]; r2 += rel[k] * rel[k]; }
        const double r = std::sqrt(r2);
        double u[3], q2 = 0.0;
        for (int k = 0; k < d; ++k) { u[k] = rel[k] * nb.ks.inv_h[k]; q2 += u[k] * u[k]; }
        const double q = std::sqrt(q2), tt = 1.0 - 0.5 * q;
        const double mag = q < 2.0 ? nb.ks.pref * (-5.0 * tt * tt * tt) : 0.0;
        double radial = 0.0;
        for (int k = 0; k < d; ++k) radial -= (rel[k] / r) * (mag * (u[k] * nb.ks.inv_h[k]));
        const double vi = d == 3 ? xv[i].w : xv[i].z, vj = d == 3 ? xv[j].w : xv[j].z;
        return 2.0 * vi * vj * radial / r;
    };
    struct ColBank {
        int row[8] = {0, 0, 0, 0, 0, 0, 0, 0}, col[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int maxrow = 0, maxcol = 0;
    };
    // MTSPH_SWEEP_BALANCE=<window>: free colours considered per pair (0 =
    // plain first-fit colouring)
    int kBalanceWindow = 8;
    if (const char *e = std::getenv("MTSPH_SWEEP_BALANCE")) kBalanceWindow = std::max(0, std::atoi(e));
    const bool balance = kBalanceWindow > 1;
    struct Cand {
        int32_t la, lb;
        int64_t a, b;
    };
    // colour the pairs by decreasing endpoint degree (MTSPH_SWEEP_ORDER=row:
    // row order): 1.381 -> 1.358 M sub-colours per pass, padding 8.5 -> 7.5 %,
    // sweep 6.20 -> 6.13 ms at 10M
    bool degree_order = true;
    if (const char *e = std::getenv("MTSPH_SWEEP_ORDER")) degree_order = std::string(e) != "row";
    auto work = [&](int64_t b0, int64_t b1) {
        std::vector<ColBank> cbank(256);
        std::vector<Cand> cand;
        std::vector<int32_t> deg;
        std::vector<std::array<uint64_t, 4>> mask;
        std::vector<int> colour;
        std::vector<std::pair<int64_t, int>> sorted_ranges;
        for (int64_t bk = b0; bk < b1; ++bk) {
            if (skip[bk]) continue;
            TaskOut &T = out[bk];
            const int64_t lo = bstart[bk], hi = bstart[bk + 1];
            int64_t cc[3] = {0, 0, 0}, bc[3] = {0, 0, 0};
            decode(cellkey[lo], d, cc);
            int col = 0;
            for (int k = d - 1; k >= 0; --k) { bc[k] = cc[k] >> lg[k]; col = col * P[k] + (int)(bc[k] % P[k]); }
            T.colour = col;
            // halo ranges: cells of the block grown by one, z-y-x order.  The
            // block owns the pairs (a, b), a < b, with a in it, so b >= lo:
            // a ring cell that lies wholly before the block in the Morton
            // order holds no partner and is left out (about half the ring)
            int local = 0;
            const int nz = d == 3 ? ext[2] + 2 : 1;
            for (int oz = 0; oz < nz; ++oz)
                for (int oy = 0; oy < ext[1] + 2; ++oy)
                    for (int ox = 0; ox < ext[0] + 2; ++ox) {
                        int64_t q[3] = {bc[0] * ext[0] - 1 + ox, bc[1] * ext[1] - 1 + oy,
                                        d == 3 ? bc[2] * ext[2] - 1 + oz : 0};
                        bool ok = true;
                        for (int k = 0; k < d; ++k) ok = ok && q[k] >= 0;
                        if (!ok) continue;
                        int64_t a, e;
                        if (!cell_range(encode(q, d), a, e)) continue;
                        if (e <= lo) continue;
                        T.ranges.push_back(make_int2((int)a, local));
                        local += (int)(e - a);
                    }
            T.halo = local;
            if (local > 65535) throw Error(1, "tiled sweep: halo too large for 16-bit local ids");
            sorted_ranges.clear();
            for (size_t r = 0; r < T.ranges.size(); ++r) sorted_ranges.emplace_back(T.ranges[r].x, (int)r);
            std::sort(sorted_ranges.begin(), sorted_ranges.end());
            auto local_of = [&](int64_t g) {
                auto it = std::upper_bound(sorted_ranges.begin(), sorted_ranges.end(),
                                           std::make_pair(g, INT32_MAX));
                --it;
                const int2 r = T.ranges[it->second];
                return r.y + (int)(g - r.x);
            };
            mask.assign(local, {0, 0, 0, 0});
            std::vector<uint32_t> pr;
            std::vector<double> pdv;
            colour.clear();
            int ncol = 0;
            for (auto &bk : cbank) bk = ColBank();
            // the block's pairs (a, b), a < b, a in the block, in row order
            cand.clear();
            for (int64_t a = lo; a < hi; ++a) {
                const int la = local_of(a);
                for (int64_t k = indptr[a]; k < indptr[a + 1]; ++k) {
                    const int64_t b = csr[k];
                    if (b <= a) continue;
                    cand.push_back({(int32_t)la, (int32_t)local_of(b), a, b});
                }
            }
            if (degree_order) {
                // colour the pairs of high-degree particles first (fewer colours)
                deg.assign(local, 0);
                for (const auto &e : cand) { ++deg[e.la]; ++deg[e.lb]; }
                std::stable_sort(cand.begin(), cand.end(), [&](const Cand &x, const Cand &y) {
                    return std::max(deg[x.la], deg[x.lb]) > std::max(deg[y.la], deg[y.lb]);
                });
            }
            for (const auto &e : cand) {
                {
                    const int la = e.la, lbb = e.lb;
                    const int64_t a = e.a, b = e.b;
                    // lowest colour free at both ends (first zero bit); with
                    // balancing, a free colour whose bank rows (li % 8) and
                    // columns (lj % 8) this pair does not push past the
                    // colour's fullest row / column (the padding bank_order
                    // needs is set by those maxima): the first such colour of
                    // each 64-colour word, words scanned while fewer than
                    // kBalanceWindow free colours have been seen, the last
                    // one found wins (else the lowest free colour).  Stopping
                    // at the first fit across words measured worse (1.43 M vs
                    // 1.36 M sub-colours, 6.27 vs 6.13 ms), as did a soft
                    // size cap preferring colours under 400-440 pairs.
                    int c = 256;
                    const int ra = la & 7, cb = lbb & 7;
                    int seen = 0;
                    for (int wd = 0; wd < 4 && seen < (balance ? kBalanceWindow : 1); ++wd) {
                        uint64_t freeb = ~(mask[la][wd] | mask[lbb][wd]);
                        while (freeb && seen < (balance ? kBalanceWindow : 1)) {
                            const int cc = wd * 64 + __builtin_ctzll(freeb);
                            freeb &= freeb - 1;
                            if (seen++ == 0) c = cc;
                            if (!balance) break;
                            const ColBank &bk = cbank[cc];
                            if (bk.row[ra] < bk.maxrow && bk.col[cb] < bk.maxcol) { c = cc; break; }
                        }
                    }
                    if (c >= 256) throw Error(1, "tiled sweep: more than 256 sub-colours");
                    if (balance) {
                        ColBank &bk = cbank[c];
                        bk.maxrow = std::max(bk.maxrow, ++bk.row[ra]);
                        bk.maxcol = std::max(bk.maxcol, ++bk.col[cb]);
                    }
                    mask[la][c >> 6] |= 1ull << (c & 63);
                    mask[lbb][c >> 6] |= 1ull << (c & 63);
                    pr.push_back((uint32_t)la | ((uint32_t)lbb << 16));
                    pdv.push_back(pdamp(a, b));
                    colour.push_back(c);
                    ncol = std::max(ncol, c + 1);
                }
            }
            // stable counting sort by sub-colour, then each sub-colour in
            // bank-conflict-free quarter-warp groups (padded)
            std::vector<int32_t> cnt(ncol + 1, 0);
            for (int c : colour) cnt[c + 1]++;
            for (int c = 0; c < ncol; ++c) cnt[c + 1] += cnt[c];
            std::vector<uint32_t> sp(pr.size());
            std::vector<double> sd(pr.size());
            std::vector<int32_t> fill(cnt.begin(), cnt.end() - 1);
            for (size_t p = 0; p < pr.size(); ++p) {
                const int w = fill[colour[p]]++;
                sp[w] = pr[p];
                sd[w] = pdv[p];
            }
            T.pairs.clear();
            T.pd.clear();
            T.sub.assign(1, 0);
            for (int c = 0; c < ncol; ++c) {
                const int32_t start = (int32_t)T.pairs.size();
                bank_order(sp.data() + cnt[c], sd.data() + cnt[c], cnt[c + 1] - cnt[c], T.pairs, T.pd);
                // whole 16 B chunks (4 pair words): every sub-colour starts 16 B
                // aligned in both streams, as the kernel's bulk copies require
                while ((T.pairs.size() - (size_t)start) % 4) {
                    T.pairs.push_back(kPadPair);
                    T.pd.push_back(0.0);
                }
                // optional cap on the sub-colour size (whole quarter-warp
                // groups): a subset of a matching is a matching, so a split
                // sub-colour is still independent pairs; smaller ring slots
                // let more CTAs share an SM
                const int32_t end = (int32_t)T.pairs.size();
                if (subcap > 0)
                    for (int32_t b = start + subcap; b < end; b += subcap) T.sub.push_back(b);
                T.sub.push_back(end);
            }
        }
    };
    const int nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    std::exception_ptr err = nullptr;
    std::mutex mu;
    const int64_t chunk = (nblocks + nth - 1) / nth;
    for (int w = 0; w < nth; ++w) {
        const int64_t b0 = w * chunk, b1 = std::min(nblocks, b0 + chunk);
        if (b0 >= b1) break;
        pool.emplace_back([&, b0, b1] {
            try { work(b0, b1); } catch (...) { std::lock_guard<std::mutex> g(mu); err = std::current_exception(); }
        });
    }
    for (auto &th : pool) th.join();
    setup_mark(s, "tiled: blocks + colouring");
    if (err) std::rethrow_exception(err);
    // colour-major task order
    int ncol = 1;
    for (int k = 0; k < d; ++k) ncol *= P[k];
    std::vector<int64_t> order;
    t.colour_ptr.assign(ncol + 1, 0);
    for (int c = 0; c < ncol; ++c) {
        for (int64_t bk = 0; bk < nblocks; ++bk) if (!skip[bk] && out[bk].colour == c) order.push_back(bk);
        t.colour_ptr[c + 1] = (int64_t)order.size();
    }
    // dataflow sweep: per task, the tasks whose halos overlap its halo (block
    // coordinates within 1, or 2 along a one-cell axis), its colour, and the
    // reverse-pass order
    {
        std::unordered_map<uint64_t, int32_t> at;
        at.reserve(order.size() * 2);
        for (size_t q = 0; q < order.size(); ++q) at[cellkey[bstart[order[q]]] >> sh] = (int32_t)q;
        std::vector<int32_t> nboff(1, 0), nbt, col(order.size()), rev;
        int r[3] = {0, 0, 0};
        for (int k = 0; k < d; ++k) r[k] = ext[k] == 1 ? 2 : 1;
        for (size_t q = 0; q < order.size(); ++q) {
            const int64_t bk = order[q];
            col[q] = out[bk].colour;
            int64_t cc[3] = {0, 0, 0}, bc[3] = {0, 0, 0};
            decode(cellkey[bstart[bk]], d, cc);
            for (int k = 0; k < d; ++k) bc[k] = cc[k] >> lg[k];
            for (int oz = -r[2]; oz <= r[2]; ++oz)
                for (int oy = -r[1]; oy <= r[1]; ++oy)
                    for (int ox = -r[0]; ox <= r[0]; ++ox) {
                        if (ox == 0 && oy == 0 && oz == 0) continue;
                        const int64_t nbc[3] = {bc[0] + ox, bc[1] + oy, bc[2] + oz};
                        if (nbc[0] < 0 || nbc[1] < 0 || nbc[2] < 0) continue;
                        const int64_t qc[3] = {nbc[0] << lg[0], nbc[1] << lg[1], nbc[2] << lg[2]};
                        auto it = at.find(encode(qc, d) >> sh);
                        if (it != at.end()) nbt.push_back(it->second);
                    }
            nboff.push_back((int32_t)nbt.size());
        }
        for (int c = ncol - 1; c >= 0; --c)
            for (int64_t q = t.colour_ptr[c]; q < t.colour_ptr[c + 1]; ++q) rev.push_back((int32_t)q);
        upload_vec(t.f_nboff, nboff, s);
        upload_vec(t.f_nbt, nbt, s);
        upload_vec(t.f_col, col, s);
        upload_vec(t.f_rev, rev, s);
        t.f_done.alloc(order.size() + 1);
    }
    setup_mark(s, "tiled: dataflow lists");
    // task-major concatenation: offsets first, then a parallel copy into
    // arrays sized once (growing multi-GB vectors cost ~8 s at 10M)
    const size_t ntk = order.size();
    std::vector<int64_t> roff(ntk + 1, 0), poff(ntk + 1, 0), soff(ntk + 1, 0);
    std::vector<int32_t> halo(ntk);
    int64_t real_pairs = 0;
    for (size_t q = 0; q < ntk; ++q) {
        const TaskOut &T = out[order[q]];
        roff[q + 1] = roff[q] + (int64_t)T.ranges.size();
        poff[q + 1] = poff[q] + (int64_t)T.pairs.size();
        soff[q + 1] = soff[q] + (int64_t)T.sub.size();
        halo[q] = T.halo;
        t.max_halo = std::max(t.max_halo, T.halo);
        t.max_ranges = std::max(t.max_ranges, (int)T.ranges.size());
        for (size_t k = 0; k + 1 < T.sub.size(); ++k) t.maxsub = std::max(t.maxsub, T.sub[k + 1] - T.sub[k]);
        // the kernel packs a sub-colour's first pair (20 bits) and count (12 bits) into one word
        if (T.pairs.size() >= (size_t(1) << 20) || t.maxsub >= (1 << 12))
            throw Error(1, "tiled sweep: block too large for the packed sub-colour bounds");
        t.max_nsub = std::max(t.max_nsub, (int)T.sub.size() - 1);
        t.nsub_total += (int64_t)T.sub.size() - 1;
    }
    std::vector<int64_t> real_part(nth, 0);
    RawVec<int2> ranges(roff[ntk]);
    RawVec<int32_t> sub(soff[ntk]);
    RawVec<uint32_t> pairs(poff[ntk]);
    RawVec<double> pd(poff[ntk]);
    {
        std::vector<std::thread> cp;
        const size_t per = (ntk + nth - 1) / nth;
        for (int w = 0; w < nth; ++w) {
            const size_t q0 = w * per, q1 = std::min(ntk, q0 + per);
            if (q0 >= q1) break;
            cp.emplace_back([&, q0, q1, w] {
                for (size_t q = q0; q < q1; ++q) {
                    TaskOut &T = out[order[q]];
                    for (uint32_t p : T.pairs) real_part[w] += p != kPadPair;
                    std::copy(T.ranges.begin(), T.ranges.end(), ranges.begin() + roff[q]);
                    std::copy(T.pairs.begin(), T.pairs.end(), pairs.begin() + poff[q]);
                    std::copy(T.pd.begin(), T.pd.end(), pd.begin() + poff[q]);
                    std::copy(T.sub.begin(), T.sub.end(), sub.begin() + soff[q]);
                    std::vector<int2>().swap(T.ranges);
                    std::vector<uint32_t>().swap(T.pairs);
                    std::vector<double>().swap(T.pd);
                }
            });
        }
        for (auto &th : cp) th.join();
        for (int64_t v : real_part) real_pairs += v;
    }
    setup_mark(s, "tiled: concatenate");
    t.sh = sh;
    t.ntasks = (int64_t)ntk;
    t.npairs = real_pairs;
    upload_vec(t.range_off, roff, s);
    upload_vec(t.ranges, ranges, s);
    upload_vec(t.halo_n, halo, s);
    {
        std::vector<int64_t> hoff(ntk + 1, 0);
        for (size_t q = 0; q < ntk; ++q) hoff[q + 1] = hoff[q] + halo[q];
        upload_vec(t.hid_off, hoff, s);
        t.hid.alloc((size_t)std::max<int64_t>(hoff[ntk], 1));
        if (ntk)
            k_tiled_halo_ids<<<(unsigned)ntk, 256, 0, s>>>(t.range_off.p, t.ranges.p, t.halo_n.p, t.hid_off.p, t.hid.p);
        MT_LAUNCH_CHECK();
    }
    upload_vec(t.pair_off, poff, s);
    upload_vec(t.pairs, pairs, s);
    upload_vec(t.pd, pd, s);
    upload_vec(t.sub_off, soff, s);
    upload_vec(t.sub, sub, s);
    setup_mark(s, "tiled: upload");
}

// Block shape: a cubic edge of `tile` cells if given (a multi-rank plan's
// edge: exact, or an error), else 4 x 4 (x 4) cells -- a ~150 KB halo in
// 3D, one 1024-thread CTA per SM with ~500 pairs per sub-colour -- losing
// one Morton bit (halving one axis) until the halo fits shared memory.
// Measured at 10M particles (3D, bar_3d): 2^3 cells / 128 threads 15.7 ms
// per sweep, 4^3 / 1024 10.5 ms.  MTSPH_TILE_BITS (low Morton bits per
// block) / MTSPH_TILE_THREADS override for tuning.
inline void build_tiled_auto(const NbhDev &nb, TiledSched &t, cudaStream_t s, int tile = 0) {
    const size_t budget = 224 * 1024;  // opt-in maximum per CTA is 227 KB
    const int d = nb.d;
    // 3D: 4^3 cells; 2D: 16^2 cells (measured, 10M 2D bar: 4^2 / 1024 thr
    // 15.3 ms per sweep, 4^2 / 256 2.9, 8^2 4.3, 16^2 2.05; larger does not fit)
    int sh0 = d == 3 ? 6 : 8, th = 0;
    if (tile > 0) {
        if (tile & (tile - 1)) throw Error(1, "tiled sweep: block edge must be a power of two");
        sh0 = 0;
        while ((1 << (sh0 / d)) < tile) sh0 += d;
    } else if (const char *e = std::getenv("MTSPH_TILE_BITS")) {
        sh0 = std::max(0, std::atoi(e));
    }
    // multiple of 64 (>= 64): whole staging warps plus whole pair warps
    if (const char *e = std::getenv("MTSPH_TILE_THREADS")) th = std::min(1024, std::max(64, std::atoi(e) & ~63));
    for (int sh = sh0; sh >= 0; --sh) {
        t = TiledSched();
        build_tiled(nb, sh, t, s);
        if (tiled_smem_bytes(t, d) <= budget) break;
        if (tile > 0) throw Error(1, "tiled sweep: halo of the requested block edge exceeds shared memory");
        if (sh == 0) throw Error(1, "tiled sweep: particle density too high for shared memory");
    }
    if (th == 0) {
        // about two threads per (padded) pair of an average sub-colour: the
        // measured optimum for 4^3 (3D, ~550 -> 1024), 16^2 (2D, ~700 ->
        // 1024) and the small fallback blocks (4^2 in 2D: 256 beat 1024 5x)
        const double avg = t.nsub_total ? (double)t.pairs.n / (double)t.nsub_total : 0.0;
        th = std::min(1024, std::max(128, ((int)(2.0 * avg) + 63) & ~63));
        // 512 threads (64 staging + 448 pair lanes, the sub-colour cap):
        // two (fp64) / three (fp32) CTAs per SM; measured (10M, 3D) 1024
        // threads with uncapped sub-colours 7.35 / 4.22 ms, 512 with the cap
        // 6.58 / 3.94 (2D 2.01 / 1.14 -> 1.78 / 1.05)
        if (!std::getenv("MTSPH_SWEEP_SUBCAP")) th = 512;
    }
    t.threads = th;
    // the attribute is per function, shared by every problem instance: allow
    // the opt-in maximum once (the launch's own size sets the occupancy)
    allow_max_dynamic_smem((const void *)k_sweep_tiled<2>);
    allow_max_dynamic_smem((const void *)k_sweep_tiled<3>);
    allow_max_dynamic_smem((const void *)k_sweep_flow<2>);
    allow_max_dynamic_smem((const void *)k_sweep_flow<3>);
    allow_max_dynamic_smem((const void *)k_sweep_tiled<2, float>);
    allow_max_dynamic_smem((const void *)k_sweep_tiled<3, float>);
    allow_max_dynamic_smem((const void *)k_sweep_flow<2, float>);
    allow_max_dynamic_smem((const void *)k_sweep_flow<3, float>);
    // persistent dataflow launch (default; MTSPH_SWEEP_FLOW=0: per-colour
    // launches): as many CTAs as fit at once
    const char *fe = std::getenv("MTSPH_SWEEP_FLOW");
    if (!(fe && fe[0] == '0')) {
        int dev = 0, sms = 0, per = 0;
        MT_CUDA(cudaGetDevice(&dev));
        MT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        MT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per, d == 3 ? (const void *)k_sweep_flow<3> : (const void *)k_sweep_flow<2>, th,
            tiled_smem_bytes(t, d)));
        t.flow_grid = sms * per;
        MT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per, d == 3 ? (const void *)k_sweep_flow<3, float> : (const void *)k_sweep_flow<2, float>, th,
            tiled_smem_bytes(t, d, 4)));
        t.flow_grid32 = sms * per;
    }
    if (const char *e = std::getenv("MTSPH_VERBOSE"); e && e[0] == '1')
        std::fprintf(stderr,
                     "[mtsph] tiled sweep: %d Morton bits/block, %lld tasks, %lld pairs in %lld slots (%.1f %% "
                     "padding), %lld sub-colours, max halo %d, max sub-colour %d, "
                     "%d threads, smem %zu B (fp64) %zu B (fp32), dataflow grid %d / %d, %d stages (fp64)\n",
                     t.sh, (long long)t.ntasks, (long long)t.npairs, (long long)t.pairs.n,
                     t.pairs.n ? 100.0 * (1.0 - (double)t.npairs / (double)t.pairs.n) : 0.0,
                     (long long)t.nsub_total, t.max_halo, t.maxsub, t.threads, tiled_smem_bytes(t, d),
                     tiled_smem_bytes(t, d, 4), t.flow_grid, t.flow_grid32, sweep_stages(8));
}

}  // namespace mtsph
