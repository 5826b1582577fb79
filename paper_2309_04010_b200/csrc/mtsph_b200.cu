// mtsph_b200.cu -- the C ABI (include/mtsph_b200.h) over the sm_100a kernels.
//
// Host runtime in C++: owns device memory, one stream per problem, CUDA
// graphs for the device-side inner loop, error translation to the
// reference's error classes.  Compiled with
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -shared
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <type_traits>
#include <string>
#include <vector>

#include "../../include/mtsph_b200.h"
#include "common.cuh"
#include "damping.cuh"
#include "nbh.cuh"
#include "porous.cuh"
#include "solid.cuh"
#include "tiled.cuh"
#include "gather_csr.cuh"
#include "window.cuh"
#include "solid32.cuh"
#include "layer1.cuh"

using namespace mtsph;

// ------------------------------------------------------------- errors

static thread_local std::string g_err;
static thread_local std::vector<int64_t> g_err_ids;

static int fail(int code, const std::string &msg, std::vector<int64_t> ids = {}) {
    g_err = msg;
    g_err_ids = std::move(ids);
    return code;
}

#define API_BEGIN try {
#define API_END                                                                \
    }                                                                          \
    catch (const mtsph::Error &e) { return fail(e.code, e.what(), e.ids); }    \
    catch (const std::exception &e) { return fail(MTSPH_ERR_CUDA, e.what()); } \
    return MTSPH_OK;

extern "C" int mtsph_abi_version(void) { return MTSPH_ABI_VERSION; }
extern "C" const char *mtsph_last_error(void) { return g_err.c_str(); }
extern "C" int64_t mtsph_last_error_ids(int64_t *ids, int64_t cap) {
    int64_t n = (int64_t)g_err_ids.size();
    for (int64_t k = 0; k < n && k < cap; ++k) ids[k] = g_err_ids[k];
    return n;
}
extern "C" int mtsph_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) { cudaGetLastError(); return 0; }
    return c;
}

// the device this library's runtime places new problems on (one process
// per GPU: the rank's local device).  The library carries its own CUDA
// runtime, so torch.cuda.set_device does not select it.
extern "C" mtsph_status mtsph_set_device(int ordinal) {
    API_BEGIN
    const int c = mtsph_device_count();
    if (ordinal < 0 || ordinal >= c)
        throw Error(MTSPH_ERR_ARG, "device ordinal " + std::to_string(ordinal) + " out of range (" +
                                       std::to_string(c) + " devices)");
    MT_CUDA(cudaSetDevice(ordinal));
    API_END
}

static void require_device() {
    if (mtsph_device_count() <= 0) throw Error(MTSPH_ERR_CUDA, "no CUDA device available");
}

// ------------------------------------------------------------- neighbourhood

struct mtsph_nbh {
    NbhDev nb;
    cudaStream_t s = nullptr;
    ~mtsph_nbh() { if (s) cudaStreamDestroy(s); }
};

extern "C" mtsph_status mtsph_nbh_create(int64_t n, int d, const double *pos, const double *vol,
                                         const double *h_axes, int sweep, mtsph_nbh **out) {
    API_BEGIN
    require_device();
    auto h = std::make_unique<mtsph_nbh>();
    MT_CUDA(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
    build_nbh(h->nb, n, d, pos, vol, h_axes, sweep, h->s);
    *out = h.release();
    API_END
}

extern "C" mtsph_status mtsph_nbh_destroy(mtsph_nbh *nb) {
    delete nb;
    return MTSPH_OK;
}

extern "C" mtsph_status mtsph_nbh_sizes(const mtsph_nbh *h, int64_t *nnz, int64_t *npairs, int64_t *ngroups,
                                        int64_t *nphases) {
    if (!h) return fail(MTSPH_ERR_ARG, "mtsph_nbh_sizes: null handle");
    const NbhDev &nb = h->nb;
    if (nnz) *nnz = nb.nnz;
    if (npairs) *npairs = nb.npairs;
    if (ngroups) *ngroups = nb.ngroups;
    if (nphases) {
        if (nb.sweep == 1) *nphases = nb.nlevels;
        else if (nb.sweep == 2) {
            int64_t c = 0;
            for (size_t k = 0; k + 1 < nb.colour_task_ptr.size(); ++k)
                c += nb.colour_task_ptr[k + 1] > nb.colour_task_ptr[k];
            *nphases = c;
        } else *nphases = 0;
    }
    return MTSPH_OK;
}

extern "C" mtsph_status mtsph_nbh_permutation(const mtsph_nbh *h, int64_t *perm) {
    if (!h) return fail(MTSPH_ERR_ARG, "mtsph_nbh_permutation: null handle");
    API_BEGIN
    h->nb.perm.download(perm, h->nb.n, h->s);
    MT_CUDA(cudaStreamSynchronize(h->s));
    API_END
}

// host-side kernel gradient identical to the device grad_w
static void grad_host(int d, const double *rel, const KSpec &ks, double *g) {
    double u[3], q2 = 0.0;
    for (int k = 0; k < d; ++k) { u[k] = rel[k] * ks.inv_h[k]; q2 += u[k] * u[k]; }
    const double q = std::sqrt(q2), t = 1.0 - 0.5 * q;
    const double mag = q < 2.0 ? ks.pref * (-5.0 * t * t * t) : 0.0;
    for (int k = 0; k < d; ++k) g[k] = mag * (u[k] * ks.inv_h[k]);
}

extern "C" mtsph_status mtsph_nbh_export(const mtsph_nbh *h, int64_t *indptr, int64_t *idx, double *grad0,
                                         int64_t *pair_i, int64_t *pair_j, double *pair_damp,
                                         double *pair_grad, int64_t *pair_group, double *corr) {
    if (!h) return fail(MTSPH_ERR_ARG, "mtsph_nbh_export: null handle");
    API_BEGIN
    const NbhDev &nb = h->nb;
    const int64_t n = nb.n;
    const int d = nb.d;
    cudaStream_t s = h->s;
    std::vector<int64_t> perm(n), iptr(n + 1);
    std::vector<int32_t> csr(std::max<int64_t>(nb.nnz, 1));
    std::vector<double4> XV(n);
    nb.perm.download(perm.data(), n, s);
    nb.indptr.download(iptr.data(), n + 1, s);
    nb.csr.download(csr.data(), nb.nnz, s);
    nb.XV.download(XV.data(), n, s);
    MT_CUDA(cudaStreamSynchronize(s));
    auto X = [&](int64_t k, int c) {
        const double4 &q = XV[k];
        return c == 0 ? q.x : (c == 1 ? q.y : q.z);
    };
    auto Vol = [&](int64_t k) { return d == 3 ? XV[k].w : XV[k].z; };
    // reference CSR: rows in original order, neighbours ascending original id
    std::vector<int64_t> iperm(n);
    for (int64_t k = 0; k < n; ++k) iperm[perm[k]] = k;
    int64_t w = 0;
    if (indptr) indptr[0] = 0;
    std::vector<std::pair<int64_t, int32_t>> row;
    for (int64_t o = 0; o < n; ++o) {
        const int64_t a = iperm[o];
        row.clear();
        for (int64_t k = iptr[a]; k < iptr[a + 1]; ++k) row.emplace_back(perm[csr[k]], csr[k]);
        std::sort(row.begin(), row.end());
        for (auto &e : row) {
            if (idx) idx[w] = e.first;
            if (grad0) {
                double rel[3];
                for (int c = 0; c < d; ++c) rel[c] = X(e.second, c) - X(a, c);
                grad_host(d, rel, nb.ks, grad0 + w * d);
            }
            ++w;
        }
        if (indptr) indptr[o + 1] = w;
    }
    if (corr) {
        std::vector<double> B((size_t)n * d * d);
        nb.B.download(B.data(), B.size(), s);
        MT_CUDA(cudaStreamSynchronize(s));
        for (int64_t k = 0; k < n; ++k)
            for (int q = 0; q < d * d; ++q) corr[perm[k] * d * d + q] = B[(size_t)q * n + k];
    }
    if (nb.sweep && nb.npairs) {
        std::vector<int32_t> pi(nb.npairs), pj(nb.npairs);
        std::vector<int64_t> gp(nb.ngroups + 1);
        nb.pi.download(pi.data(), nb.npairs, s);
        nb.pj.download(pj.data(), nb.npairs, s);
        nb.gptr.download(gp.data(), nb.ngroups + 1, s);
        MT_CUDA(cudaStreamSynchronize(s));
        // export in execution order: SERIAL = reference order; COLOURED =
        // colour-major, task order
        for (int64_t k = 0; k < nb.npairs; ++k) {
            if (pair_i) pair_i[k] = perm[pi[k]];
            if (pair_j) pair_j[k] = perm[pj[k]];
            double rel[3], g[3], r2 = 0.0;
            for (int c = 0; c < d; ++c) { rel[c] = X(pj[k], c) - X(pi[k], c); r2 += rel[c] * rel[c]; }
            grad_host(d, rel, nb.ks, g);
            if (pair_grad) for (int c = 0; c < d; ++c) pair_grad[k * d + c] = g[c];
            if (pair_damp) {
                const double r = std::sqrt(r2);
                double radial = 0.0;
                for (int c = 0; c < d; ++c) radial -= (rel[c] / r) * g[c];
                pair_damp[k] = 2.0 * Vol(pi[k]) * Vol(pj[k]) * radial / r;
            }
        }
        if (pair_group) for (int64_t g = 0; g <= nb.ngroups; ++g) pair_group[g] = gp[g];
    } else if (pair_group) {
        pair_group[0] = 0;
    }
    API_END
}

// ------------------------------------------------------------- solid

struct mtsph_solid {
    NbhDev nb;
    int d = 0;
    int64_t n = 0;
    cudaStream_t s = nullptr;
    DBuf<unsigned char> V;
    DBuf<double> x, a, F, cp, alpha, T, G, mass, rho0, inv_m, part, meas;
    DBuf<uint8_t> flags;
    DBuf<Ctrl> ctrl;
    DBuf<int64_t> level_ptr;
    TiledSched tiled;
    std::vector<int64_t> iperm_h;  // original -> internal (lazy, for pack/unpack)
    // 0: SELL gathers; G: row-parallel CSR gathers, G lanes per particle.
    // Measured (10M, 3D): SELL 7.4 + 10.0 ms, G=2 5.8 + 7.4, G=4 5.8 + 7.3,
    // G=8 6.9 + 8.7 (stress + accel); MTSPH_GATHER_LANES overrides
    int gather_g = 4;
    // passes per wide gather CTA (0: the 256-thread kernels); set at setup from
    // the particle count, MTSPH_ACCEL_WIDE / MTSPH_STRESS_WIDE override (0, 2, 4, 8 / 0, 4)
    int accel_np = 0, stress_np = 0;
    // 3D fp64 opt-in (MTSPH_GATHER_WINDOW=1): shared-memory cell-window
    // gathers (window.cuh; measured slower than the CSR gathers)
    WinSched win;
    DBuf<double> Lacc;  // its stress sums, [d*d][n]
    Ctrl *hc = nullptr;  // pinned mirror
    Mat mat{};
    int nblk = 0;
    int64_t launches = 0;
    int per_step_launches = 0;
    cudaGraphExec_t graphs[3] = {nullptr, nullptr, nullptr};
    int graph_steps[3] = {4, 32, 128};
    // fp32 variant (solid32.cuh): prec 32 = the fp32 arrays below hold the
    // state and the fp64 ones are a mirror, refreshed whenever the host reads
    // them (a steps counter cannot tell: steps also run inside CUDA graphs)
    int prec = 64;
    int gather_g32 = 4;  // lanes per particle of the fp32 gathers (MTSPH_GATHER_LANES32)
    DBuf<float> XV32, B32, G32, mass32, rho032, inv_m32, pd32, u32, a32, H32, Hc32, alpha32, T32;
    DBuf<unsigned char> V32;
    TiledArgsT<float> tiled_args32() {
        TiledArgsT<float> A{tiled.range_off.p, tiled.ranges.p, tiled.halo_n.p, tiled.pair_off.p, tiled.pairs.p,
                            pd32.p, tiled.sub_off.p, tiled.sub.p, inv_m32.p, V32.p, tiled.maxsub,
                            tiled.hid_off.p, tiled.hid.p};
        return A;
    }
    Solid32Args args32() {
        Solid32Args A{};
        A.n = n;
        A.XV = reinterpret_cast<const float4 *>(XV32.p);
        A.V = V32.p;
        A.u = u32.p; A.a = a32.p; A.H = H32.p; A.Hc = Hc32.p; A.alpha = alpha32.p; A.T = T32.p;
        A.B = B32.p; A.G = G32.p; A.mass = mass32.p; A.rho0 = rho032.p; A.flags = flags.p;
        A.indptr = nb.indptr.p; A.csr = nb.csr.p;
        A.cptr = nb.chunk_g ? nb.cptr.p : nullptr; A.csr16 = nb.csr16.p;
        A.perm = nb.perm.p;
        A.part = part.p;
        A.nblk = nblk;
        A.ctrl = ctrl.p;
        A.ks = kspec32(nb.ks);
        A.mat = mat;
        return A;
    }
    void drop_graphs() {
        for (auto &g : graphs) if (g) { cudaGraphExecDestroy(g); g = nullptr; }
    }
    TiledArgs tiled_args() {
        TiledArgs A{tiled.range_off.p, tiled.ranges.p, tiled.halo_n.p, tiled.pair_off.p, tiled.pairs.p,
                    tiled.pd.p, tiled.sub_off.p, tiled.sub.p, inv_m.p, V.p, tiled.maxsub, tiled.hid_off.p, tiled.hid.p};
        return A;
    }
    ~mtsph_solid() {
        for (auto &g : graphs) if (g) cudaGraphExecDestroy(g);
        if (hc) cudaFreeHost(hc);
        if (s) cudaStreamDestroy(s);
    }
    SolidArgs args() {
        SolidArgs A{};
        A.n = n;
        A.XV = nb.XV.p;
        A.V = V.p;
        A.x = x.p; A.a = a.p; A.F = F.p; A.cp = cp.p; A.alpha = alpha.p; A.T = T.p;
        A.B = nb.B.p; A.G = G.p; A.mass = mass.p; A.rho0 = rho0.p; A.flags = flags.p;
        A.slice_ptr = nb.slice_ptr.p; A.slice_w = nb.slice_w.p; A.nbr = nb.nbr.p;
        A.indptr = nb.indptr.p; A.csr = nb.csr.p;
        A.cptr = nb.chunk_g ? nb.cptr.p : nullptr; A.csr16 = nb.csr16.p; A.mag16 = nb.mag16.p;
        A.perm = nb.perm.p;
        A.Lacc = win.on ? Lacc.p : nullptr;
        A.part = part.p;
        A.nblk = nblk;
        A.ctrl = ctrl.p;
        A.ks = nb.ks;
        A.mat = mat;
        return A;
    }
    SweepArgs sweep_args() {
        SweepArgs S{};
        S.pi = nb.pi.p; S.pj = nb.pj.p; S.gptr = nb.gptr.p; S.gscr = nb.gscr.p;
        S.scratch = nb.scratch.p; S.XV = nb.XV.p; S.inv_m = inv_m.p; S.V = V.p; S.ks = nb.ks;
        return S;
    }
    void pull_ctrl() {
        MT_CUDA(cudaMemcpyAsync(hc, ctrl.p, sizeof(Ctrl), cudaMemcpyDeviceToHost, s));
        MT_CUDA(cudaStreamSynchronize(s));
    }
    void push_ctrl() {
        MT_CUDA(cudaMemcpyAsync(ctrl.p, hc, sizeof(Ctrl), cudaMemcpyHostToDevice, s));
        MT_CUDA(cudaStreamSynchronize(s));
    }
};

// neighbour gathers: row-parallel CSR (default, gather_g lanes per particle),
// SELL (gather_g = 0), or block-tiled shared memory (opt-in, slower)
// (returns the number of kernels launched)
template <int D> static int launch_stress_gather(mtsph_solid *S, const SolidArgs &A, cudaStream_t s) {
    const unsigned nb = blocks_for(S->n);
    if (D == 3 && S->win.on) {
        if (S->win.ntasks > 0)
            k_win_stress<<<(unsigned)S->win.ntasks, S->win.threads, win_smem(S->win, 2, 9), s>>>(A, win_args(S->win, S->nb));
        return 1;
    }
    const bool c16 = S->nb.chunk_g == S->gather_g && S->gather_g > 0;
    if (S->gather_g == 4 && c16 && A.mag16 && S->stress_np == 4) k_solid_stress_csr<D, 4, true, true, 4, 4><<<(unsigned)((S->n + 4095) / 4096), 1024, 0, s>>>(A);
    else if (S->gather_g == 4 && c16 && A.mag16) k_solid_stress_csr<D, 4, true, true><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 4 && c16) k_solid_stress_csr<D, 4, true><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 2 && c16) k_solid_stress_csr<D, 2, true><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 4) k_solid_stress_csr<D, 4><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 8) k_solid_stress_csr<D, 8><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 2) k_solid_stress_csr<D, 2><<<nb, 256, 0, s>>>(A);
    else k_solid_stress<D, true><<<nb, 256, 0, s>>>(A);
    return 1;
}
// the split return map, instantiated per hardening law
template <int D> static void launch_rmap(mtsph_solid *S, const SolidArgs &A, cudaStream_t s) {
    const unsigned nb = blocks_for(S->n);
    if (S->mat.law == 1) k_solid_rmap<D, 1><<<nb, 256, 0, s>>>(A);
    else k_solid_rmap<D, 0><<<nb, 256, 0, s>>>(A);
}
template <int D> static int launch_accel_gather(mtsph_solid *S, const SolidArgs &A, cudaStream_t s) {
    const unsigned nb = blocks_for(S->n);
    if (D == 3 && S->win.on) {
        if (S->win.ntasks > 0)
            k_win_accel<<<(unsigned)S->win.ntasks, S->win.threads, win_smem(S->win, 3, 3), s>>>(A, win_args(S->win, S->nb));
        k_solid_kick_part<D><<<nb, 256, 0, s>>>(A);
        return 2;
    }
    const bool c16 = S->nb.chunk_g == S->gather_g && S->gather_g > 0;
    // (the stored gradient magnitudes cost the divergence gather registers: 5.27 -> 5.45 ms)
    // large problems: one 768-thread CTA per SM working through 768 NP
    // particles 192 consecutive ones at a time (gather_csr.cuh); accel_np is
    // chosen at setup so that the grid still has several waves
    const int anp = S->accel_np;
    if (S->gather_g == 4 && c16 && anp == 8) k_solid_accel_csr<D, 4, true, false, 3, 8><<<(unsigned)((S->n + 6143) / 6144), 768, 0, s>>>(A);
    else if (S->gather_g == 4 && c16 && anp == 4) k_solid_accel_csr<D, 4, true, false, 3, 4><<<(unsigned)((S->n + 3071) / 3072), 768, 0, s>>>(A);
    else if (S->gather_g == 4 && c16 && anp == 2) k_solid_accel_csr<D, 4, true, false, 3, 2><<<(unsigned)((S->n + 1535) / 1536), 768, 0, s>>>(A);
    else if (S->gather_g == 4 && c16) k_solid_accel_csr<D, 4, true><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 2 && c16) k_solid_accel_csr<D, 2, true><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 4) k_solid_accel_csr<D, 4><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 8) k_solid_accel_csr<D, 8><<<nb, 256, 0, s>>>(A);
    else if (S->gather_g == 2) k_solid_accel_csr<D, 2><<<nb, 256, 0, s>>>(A);
    else k_solid_accel<D><<<nb, 256, 0, s>>>(A);
    return 1;
}

// one inner step; ev (optional, 6 events) brackets the kernel classes
template <int D> static int solid_step(mtsph_solid *S, int ctrl_mode, cudaEvent_t *ev = nullptr) {
    SolidArgs A = S->args();
    const unsigned nb = blocks_for(S->n);
    // external record: under stream capture this becomes an event-record
    // node of the graph (a plain record would only order the capture)
    auto mark = [&](int k) { if (ev) MT_CUDA(cudaEventRecordWithFlags(ev[k], S->s, cudaEventRecordExternal)); };
    mark(0);
    k_solid_kick_drift<D><<<nb, 256, 0, S->s>>>(A);
    mark(1);
    // split: the neighbour gather runs at low register count / high
    // occupancy, the register-heavy return map element-wise
    int extra = launch_stress_gather<D>(S, A, S->s) - 1;
    launch_rmap<D>(S, A, S->s);
    mark(2);
    extra += launch_accel_gather<D>(S, A, S->s) - 1;
    MT_LAUNCH_CHECK();
    mark(3);
    int l = 3 + extra + (S->nb.sweep == 3 ? launch_tiled_sweep<D>(S->tiled, S->tiled_args(), S->ctrl.p, S->s)
                                   : launch_sweep<D>(S->nb, S->sweep_args(), S->level_ptr.p, S->ctrl.p, S->s));
    mark(4);
    k_solid_vmax<D><<<nb, 256, 0, S->s>>>(A, 0);
    k_ctrl<<<1, kCtrlThreads, 0, S->s>>>(S->ctrl.p, S->part.p, S->nblk, ctrl_mode);
    MT_LAUNCH_CHECK();
    mark(5);
    return l + 2;
}

// the fp32 variant of solid_step (solid32.cuh): same kernel classes and
// event marks, row-parallel gathers with 4 lanes per particle, tiled sweep
template <int D> static int solid_step32(mtsph_solid *S, int ctrl_mode, cudaEvent_t *ev = nullptr) {
    Solid32Args A = S->args32();
    const unsigned nb = blocks_for(S->n);
    auto mark = [&](int k) { if (ev) MT_CUDA(cudaEventRecordWithFlags(ev[k], S->s, cudaEventRecordExternal)); };
    mark(0);
    k32_kick_drift<D><<<nb, 256, 0, S->s>>>(A);
    mark(1);
    const bool c16 = S->nb.chunk_g == S->gather_g32;
    switch (c16 ? -S->gather_g32 : S->gather_g32) {
    case -2: k32_stress_csr<D, 2, true><<<nb, 256, 0, S->s>>>(A); break;
    case -4: k32_stress_csr<D, 4, true><<<nb, 256, 0, S->s>>>(A); break;
    case 2: k32_stress_csr<D, 2><<<nb, 256, 0, S->s>>>(A); break;
    case 8: k32_stress_csr<D, 8><<<nb, 256, 0, S->s>>>(A); break;
    case 16: k32_stress_csr<D, 16><<<nb, 256, 0, S->s>>>(A); break;
    default: k32_stress_csr<D, 4><<<nb, 256, 0, S->s>>>(A);
    }
    if (S->mat.law == 1) k32_rmap<D, 1><<<nb, 256, 0, S->s>>>(A);
    else k32_rmap<D, 0><<<nb, 256, 0, S->s>>>(A);
    mark(2);
    switch (c16 ? -S->gather_g32 : S->gather_g32) {
    case -2: k32_accel_csr<D, 2, true><<<nb, 256, 0, S->s>>>(A); break;
    case -4: k32_accel_csr<D, 4, true><<<nb, 256, 0, S->s>>>(A); break;
    case 2: k32_accel_csr<D, 2><<<nb, 256, 0, S->s>>>(A); break;
    case 8: k32_accel_csr<D, 8><<<nb, 256, 0, S->s>>>(A); break;
    case 16: k32_accel_csr<D, 16><<<nb, 256, 0, S->s>>>(A); break;
    default: k32_accel_csr<D, 4><<<nb, 256, 0, S->s>>>(A);
    }
    MT_LAUNCH_CHECK();
    mark(3);
    int l = 3 + launch_tiled_sweep<D, float>(S->tiled, S->tiled_args32(), S->ctrl.p, S->s);
    mark(4);
    k32_vmax<D><<<nb, 256, 0, S->s>>>(A, 0);
    k_ctrl<<<1, kCtrlThreads, 0, S->s>>>(S->ctrl.p, S->part.p, S->nblk, ctrl_mode);
    MT_LAUNCH_CHECK();
    mark(5);
    return l + 2;
}

static int solid_step_any(mtsph_solid *S, int mode, cudaEvent_t *ev = nullptr) {
    if (S->prec == 32) return S->d == 2 ? solid_step32<2>(S, mode, ev) : solid_step32<3>(S, mode, ev);
    return S->d == 2 ? solid_step<2>(S, mode, ev) : solid_step<3>(S, mode, ev);
}

template <int D> static void solid_init_dt(mtsph_solid *S) {
    if (S->prec == 32) k32_vmax<D><<<blocks_for(S->n), 256, 0, S->s>>>(S->args32(), 1);
    else k_solid_vmax<D><<<blocks_for(S->n), 256, 0, S->s>>>(S->args(), 1);
    k_ctrl<<<1, kCtrlThreads, 0, S->s>>>(S->ctrl.p, S->part.p, S->nblk, CTRL_INIT);
    MT_LAUNCH_CHECK();
    S->launches += 2;
}

static void g_timed_reset();
static void g_timed_drop(const mtsph_solid *owner);

// fp32 state -> the fp64 mirror (before anything reads the fp64 arrays)
static void sync64(mtsph_solid *S) {
    if (S->prec != 32) return;
    const unsigned nb = blocks_for(S->n);
    if (S->d == 2) k32_convert<2><<<nb, 256, 0, S->s>>>(S->args(), S->args32(), 0);
    else k32_convert<3><<<nb, 256, 0, S->s>>>(S->args(), S->args32(), 0);
    MT_LAUNCH_CHECK();
    S->launches += 1;
}
// the fp64 arrays -> the fp32 state (after the host wrote the fp64 ones)
static void sync32(mtsph_solid *S) {
    if (S->prec != 32) return;
    const unsigned nb = blocks_for(S->n);
    if (S->d == 2) k32_convert<2><<<nb, 256, 0, S->s>>>(S->args(), S->args32(), 1);
    else k32_convert<3><<<nb, 256, 0, S->s>>>(S->args(), S->args32(), 1);
    MT_LAUNCH_CHECK();
    S->launches += 1;
}

extern "C" mtsph_status mtsph_solid_set_precision(mtsph_solid *S, int bits) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_set_precision: null handle");
    API_BEGIN
    if (bits != 32 && bits != 64) throw Error(MTSPH_ERR_ARG, "precision must be 32 or 64 bits");
    if (bits == S->prec) return MTSPH_OK;
    if (bits == 32) {
        if (S->nb.sweep != 3) throw Error(MTSPH_ERR_ARG, "the fp32 variant needs the tiled sweep");
        if (!S->nb.ghost_internal.empty()) throw Error(MTSPH_ERR_ARG, "the fp32 variant is single-domain only");
        const int64_t n = S->n;
        const int d = S->d;
        if (!S->u32.p) {
            S->XV32.alloc((size_t)4 * n);
            S->B32.alloc((size_t)d * d * n);
            S->G32.alloc((size_t)d * n);
            S->mass32.alloc(n);
            S->rho032.alloc(n);
            S->inv_m32.alloc(n);
            S->pd32.alloc(std::max<size_t>(S->tiled.pd.n, 1));
            S->u32.alloc((size_t)d * n);
            S->a32.alloc((size_t)d * n);
            S->H32.alloc((size_t)d * d * n);
            S->Hc32.alloc((size_t)d * d * n);
            S->alpha32.alloc(n);
            S->T32.alloc((size_t)n * (d == 3 ? DS<3>::n : DS<2>::n));
            S->T32.zero(S->s);
            S->V32.alloc((size_t)n * (d == 3 ? sizeof(float4) : sizeof(float2)));
            const unsigned nb = blocks_for(n);
            if (d == 2) k32_static<2><<<nb, 256, 0, S->s>>>(S->args(), S->args32(), S->inv_m.p, S->inv_m32.p);
            else k32_static<3><<<nb, 256, 0, S->s>>>(S->args(), S->args32(), S->inv_m.p, S->inv_m32.p);
            const int64_t np = (int64_t)S->tiled.pd.n;
            if (np > 0) k32_narrow<<<blocks_for(np), 256, 0, S->s>>>(S->tiled.pd.p, S->pd32.p, np);
            MT_LAUNCH_CHECK();
            S->launches += np > 0 ? 2 : 1;
        }
        if (const char *e = std::getenv("MTSPH_GATHER_LANES32")) {
            const int g = std::atoi(e);
            if (g != 2 && g != 4 && g != 8 && g != 16) throw Error(MTSPH_ERR_ARG, "MTSPH_GATHER_LANES32: 2, 4, 8 or 16");
            S->gather_g32 = g;
        }
        S->prec = 32;
        sync32(S);
    } else {
        sync64(S);
        S->prec = 64;
    }
    S->drop_graphs();
    g_timed_reset();
    MT_CUDA(cudaStreamSynchronize(S->s));
    API_END
}

extern "C" mtsph_status mtsph_solid_precision(const mtsph_solid *S, int *bits) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_precision: null handle");
    *bits = S->prec;
    return MTSPH_OK;
}

static void check_solid_errors(mtsph_solid *S) {
    if (S->hc->err_inv != ~0ull)
        throw Error(MTSPH_ERR_INVERSION, "non-positive deformation determinant (first id " +
                                             std::to_string(S->hc->err_inv) + ")",
                    {(int64_t)S->hc->err_inv});
    if (S->hc->err_rm != ~0ull)
        throw Error(MTSPH_ERR_RETURN_MAP, "return mapping did not converge (first id " +
                                              std::to_string(S->hc->err_rm) + ")",
                    {(int64_t)S->hc->err_rm});
    if (S->hc->remote_err)
        throw Error(MTSPH_ERR_NONFINITE, "inner loop stopped by an error on another rank");
}

extern "C" mtsph_status mtsph_solid_create(const mtsph_solid_desc *dsc, mtsph_solid **out) {
    API_BEGIN
    require_device();
    const int64_t n = dsc->n;
    const int d = dsc->d;
    if (d != 2 && d != 3) throw Error(MTSPH_ERR_ARG, "solid problems support d = 2 or 3");
    auto S = std::make_unique<mtsph_solid>();
    S->n = n;
    S->d = d;
    MT_CUDA(cudaStreamCreateWithFlags(&S->s, cudaStreamNonBlocking));
    setup_mark(S->s, "solid: start");
    if (dsc->grid) {
        S->nb.has_grid = true;
        for (int k = 0; k < 3; ++k) {
            S->nb.grid_lo[k] = dsc->grid[k];
            S->nb.grid_hi[k] = dsc->grid[3 + k];
        }
    }
    // lanes per particle: 4 in 3D (~78 neighbours), 2 in 2D (~21):
    // measured 2D 10M fp64 4.99 -> 4.94 ms/step, fp32 3.14 -> 2.95
    S->gather_g = d == 2 ? 2 : 4;
    S->gather_g32 = d == 2 ? 2 : 4;
    if (const char *e = std::getenv("MTSPH_GATHER_LANES")) {
        const int g = std::atoi(e);
        if (g != 0 && g != 2 && g != 4 && g != 8) throw Error(MTSPH_ERR_ARG, "MTSPH_GATHER_LANES: 0, 2, 4 or 8");
        S->gather_g = g;
    }
    S->nb.want_sell = S->gather_g == 0;
    if (dsc->ghost && dsc->sweep != 3 && dsc->sweep != 0)
        throw Error(MTSPH_ERR_ARG, "ghost particles (multi-rank) need the tiled sweep");
    if (dsc->ghost) {
        // ghost flags in the internal order are needed by the tiled
        // schedule; the neighbour build fixes that order, so build it first
        // with the schedule deferred
        S->nb.ghost_orig = dsc->ghost;
        build_nbh(S->nb, n, d, dsc->pos, dsc->vol, dsc->h_axes, 0, S->s);
        S->nb.ghost_orig = nullptr;
        S->nb.sweep = dsc->sweep;
        std::vector<int64_t> pm(n);
        S->nb.perm.download(pm.data(), n, S->s);
        MT_CUDA(cudaStreamSynchronize(S->s));
        S->nb.ghost_internal.resize(n);
        for (int64_t k = 0; k < n; ++k) S->nb.ghost_internal[k] = dsc->ghost[pm[k]] ? 1 : 0;
    } else {
        build_nbh(S->nb, n, d, dsc->pos, dsc->vol, dsc->h_axes, dsc->sweep, S->s);
    }
    setup_mark(S->s, "neighbourhood");
    if (S->gather_g == 2 || S->gather_g == 4) build_chunked(S->nb, S->gather_g, S->s, false, S->gather_g == 4);
    setup_mark(S->s, "chunked index table");
    if (dsc->sweep == 3) build_tiled_auto(S->nb, S->tiled, S->s, dsc->tile);
    setup_mark(S->s, "tiled schedule");
    // window gathers when asked for (MTSPH_GATHER_WINDOW=1, no CSR / SELL lane count set)
    if (d == 3 && !std::getenv("MTSPH_GATHER_LANES")) build_window(S->nb, S->win, S->s);
    if (S->win.on) S->Lacc.alloc((size_t)d * d * n);
    setup_mark(S->s, "window gathers");
    std::vector<int64_t> perm(n);
    S->nb.perm.download(perm.data(), n, S->s);
    MT_CUDA(cudaStreamSynchronize(S->s));
    const int dd = d * d;
    std::vector<double> x((size_t)d * n), F((size_t)dd * n, 0.0), mass(n), rho0(n), inv_m(n);
    std::vector<uint8_t> flags(n);
    for (int64_t k = 0; k < n; ++k) {
        const int64_t o = perm[k];
        for (int c = 0; c < d; ++c) x[(size_t)c * n + k] = dsc->pos[o * d + c];
        for (int c = 0; c < d; ++c) F[(size_t)(c * d + c) * n + k] = 1.0;
        rho0[k] = dsc->rho0[o];
        mass[k] = dsc->rho0[o] * dsc->vol[o];
        const bool movable = !dsc->constrained[o];
        inv_m[k] = movable ? 1.0 / mass[k] : 0.0;
        uint8_t f = movable ? FL_MOVABLE : 0;
        if (dsc->side && dsc->side[o] < 0) f |= FL_LEFT;
        if (dsc->side && dsc->side[o] > 0) f |= FL_RIGHT;
        if (dsc->mid_mask && dsc->mid_mask[o]) f |= FL_MID;
        if (dsc->ghost && dsc->ghost[o]) f |= FL_GHOST;
        flags[k] = f;
    }
    const size_t vbytes = (size_t)n * (d == 3 ? sizeof(double4) : sizeof(double2));
    S->V.alloc(vbytes);
    S->V.zero(S->s);
    S->x.upload(x.data(), x.size(), S->s);
    S->a.alloc((size_t)d * n);
    S->a.zero(S->s);
    S->F.upload(F.data(), F.size(), S->s);
    S->cp.upload(F.data(), F.size(), S->s);
    S->alpha.alloc(n);
    S->alpha.zero(S->s);
    S->T.alloc((size_t)n * (d == 3 ? DS<3>::n : DS<2>::n));
    S->T.zero(S->s);
    S->mass.upload(mass.data(), n, S->s);
    S->rho0.upload(rho0.data(), n, S->s);
    S->inv_m.upload(inv_m.data(), n, S->s);
    S->flags.upload(flags.data(), n, S->s);
    S->nblk = (int)blocks_for(n);
    S->G.alloc((size_t)d * n);  // static sum_b V_b gradW_ab
    if (d == 2) k_solid_gsum<2><<<blocks_for(n), 256, 0, S->s>>>(S->args(), S->G.p);
    else k_solid_gsum<3><<<blocks_for(n), 256, 0, S->s>>>(S->args(), S->G.p);
    MT_LAUNCH_CHECK();
    S->part.alloc((size_t)3 * S->nblk);
    S->part.zero(S->s);
    if (d == 3 && S->gather_g == 4) {
        // wide gather CTAs need several waves of them: >= 8 CTAs per SM
        int dev = 0, sms = 0;
        MT_CUDA(cudaGetDevice(&dev));
        MT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        const int64_t per_sm = n / std::max(sms, 1);
        S->accel_np = per_sm >= 8 * 6144 ? 8 : per_sm >= 8 * 3072 ? 4 : per_sm >= 8 * 1536 ? 2 : 0;
        S->stress_np = per_sm >= 8 * 4096 ? 4 : 0;
        if (const char *e = std::getenv("MTSPH_ACCEL_WIDE")) {
            const int v = std::atoi(e);
            if (v != 0 && v != 2 && v != 4 && v != 8) throw Error(MTSPH_ERR_ARG, "MTSPH_ACCEL_WIDE: 0, 2, 4 or 8");
            S->accel_np = v;
        }
        if (const char *e = std::getenv("MTSPH_STRESS_WIDE")) {
            const int v = std::atoi(e);
            if (v != 0 && v != 4) throw Error(MTSPH_ERR_ARG, "MTSPH_STRESS_WIDE: 0 or 4");
            S->stress_np = v;
        }
    }
    S->meas.alloc((size_t)5 * S->nblk);
    if (S->nb.sweep == 1) {
        S->level_ptr.upload(S->nb.level_ptr_h.data(), S->nb.level_ptr_h.size(), S->s);
        if (d == 2) build_serial_entries<2>(S->nb, S->sweep_args(), S->s);
        else build_serial_entries<3>(S->nb, S->sweep_args(), S->s);
    }
    Mat &m = S->mat;
    m.mu = dsc->shear_modulus;
    m.K = dsc->bulk_modulus;
    for (int k = 0; k < 4; ++k) m.p[k] = dsc->hard[k];
    m.law = dsc->hardening_law;
    m.plastic = dsc->plastic ? 1 : 0;
    m.tol = dsc->rm_tol > 0 ? dsc->rm_tol : 1e-8 * dsc->hard[0];
    m.max_iter = dsc->rm_max_iter > 0 ? dsc->rm_max_iter : 50;
    MT_CUDA(cudaMallocHost(&S->hc, sizeof(Ctrl)));
    std::memset(S->hc, 0, sizeof(Ctrl));
    S->hc->h = S->nb.ks.h_min;
    S->hc->sound = std::sqrt(dsc->bulk_modulus / dsc->rho0[0]);
    S->hc->cfl = 0.6;
    S->hc->min_dt = INFINITY;
    S->hc->err_inv = S->hc->err_rm = ~0ull;
    S->hc->remote_err = 0;
    S->hc->vol_movable = 0.0;
    S->ctrl.alloc(1);
    S->push_ctrl();
    setup_mark(S->s, "state");
    *out = S.release();
    API_END
}

extern "C" mtsph_status mtsph_solid_destroy(mtsph_solid *s) {
    g_timed_drop(s);
    delete s;
    return MTSPH_OK;
}

extern "C" mtsph_status mtsph_solid_set_ramp(mtsph_solid *S, double end_disp, int64_t ramp_steps,
                                             int64_t ramp_left) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_set_ramp: null handle");
    API_BEGIN
    S->pull_ctrl();
    S->hc->ramp_disp = end_disp / (double)(ramp_steps > 0 ? ramp_steps : 1);
    S->hc->ramp_left = ramp_left;
    S->push_ctrl();
    API_END
}

extern "C" mtsph_status mtsph_solid_ramp_left(const mtsph_solid *S, int64_t *ramp_left) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_ramp_left: null handle");
    API_BEGIN
    const_cast<mtsph_solid *>(S)->pull_ctrl();
    *ramp_left = S->hc->ramp_left;
    API_END
}

extern "C" mtsph_status mtsph_solid_stable_dt(mtsph_solid *S, double cfl, double *dt) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_stable_dt: null handle");
    API_BEGIN
    S->pull_ctrl();
    S->hc->cfl = cfl;
    S->push_ctrl();
    if (S->d == 2) solid_init_dt<2>(S); else solid_init_dt<3>(S);
    S->pull_ctrl();
    *dt = S->hc->dt;
    API_END
}

extern "C" mtsph_status mtsph_solid_relax_step(mtsph_solid *S, double dt, double eta, double *ek) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_relax_step: null handle");
    API_BEGIN
    S->pull_ctrl();
    S->hc->dt = dt;
    S->hc->eta = eta;
    S->hc->done = 0;
    S->push_ctrl();
    S->launches += solid_step_any(S, CTRL_SINGLE);
    S->pull_ctrl();
    check_solid_errors(S);
    *ek = S->hc->ek;
    API_END
}

static cudaGraphExec_t solid_graph(mtsph_solid *S, int which) {
    if (S->graphs[which]) return S->graphs[which];
    cudaGraph_t g;
    MT_CUDA(cudaStreamBeginCapture(S->s, cudaStreamCaptureModeThreadLocal));
    int l = 0;
    for (int k = 0; k < S->graph_steps[which]; ++k) l = solid_step_any(S, CTRL_STEP);
    MT_CUDA(cudaStreamEndCapture(S->s, &g));
    MT_CUDA(cudaGraphInstantiate(&S->graphs[which], g, 0));
    cudaGraphDestroy(g);
    S->per_step_launches = l;
    return S->graphs[which];
}

extern "C" mtsph_status mtsph_solid_relax(mtsph_solid *S, const mtsph_inner_params *p, mtsph_inner_result *r) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_relax: null handle");
    API_BEGIN
    S->pull_ctrl();
    Ctrl *c = S->hc;
    c->eta = p->eta;
    c->cfl = p->cfl;
    c->criterion = p->criterion;
    c->dt_outer = p->dt_outer;
    c->max_inner = p->max_inner;
    c->min_inner = p->min_inner < 1 ? 1 : p->min_inner;
    c->n_inner = 0;
    c->done = 0;
    c->cap_hit = 0;
    c->min_dt = INFINITY;
    c->err_inv = c->err_rm = ~0ull;
    c->remote_err = 0;
    S->push_ctrl();
    if (S->d == 2) solid_init_dt<2>(S); else solid_init_dt<3>(S);
    int which = 0;
    while (true) {
        cudaGraphExec_t g = solid_graph(S, which);
        MT_CUDA(cudaGraphLaunch(g, S->s));
        S->launches += (int64_t)S->graph_steps[which] * S->per_step_launches;
        S->pull_ctrl();
        if (c->done) break;
        if (which < 2) ++which;
    }
    check_solid_errors(S);
    r->n_inner = c->n_inner;
    r->cap_hit = c->cap_hit;
    r->ek = c->ek;
    r->min_dt = c->min_dt;
    r->last_dt = c->last_dt;
    API_END
}

// benchmark path: exactly nsteps steps in one graph, events per kernel class
struct TimedGraph {
    int64_t steps = 0;
    const mtsph_solid *owner = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaEvent_t> ev;
    int per_step = 0;
    ~TimedGraph() {
        if (exec) cudaGraphExecDestroy(exec);
        for (auto e : ev) cudaEventDestroy(e);
    }
};
static std::unique_ptr<TimedGraph> g_timed;  // one benchmark graph at a time
static void g_timed_reset() { g_timed.reset(); }
static void g_timed_drop(const mtsph_solid *owner) {
    if (g_timed && g_timed->owner == owner) g_timed.reset();
}

extern "C" mtsph_status mtsph_solid_run_steps(mtsph_solid *S, const mtsph_inner_params *p, int64_t nsteps,
                                              double timing[7]) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_run_steps: null handle");
    API_BEGIN
    if (nsteps <= 0) throw Error(MTSPH_ERR_ARG, "nsteps must be positive");
    S->pull_ctrl();
    Ctrl *c = S->hc;
    c->eta = p->eta;
    c->cfl = p->cfl;
    c->criterion = -1.0;          // never converged: run exactly nsteps
    c->dt_outer = p->dt_outer;
    c->max_inner = nsteps;
    c->min_inner = nsteps;
    c->n_inner = 0;
    c->done = 0;
    c->cap_hit = 0;
    c->min_dt = INFINITY;
    c->err_inv = c->err_rm = ~0ull;
    c->remote_err = 0;
    S->push_ctrl();
    if (!g_timed || g_timed->steps != nsteps || g_timed->owner != S) {
        g_timed = std::make_unique<TimedGraph>();
        g_timed->steps = nsteps;
        g_timed->owner = S;
        g_timed->ev.resize((size_t)nsteps * 6);
        for (auto &e : g_timed->ev) MT_CUDA(cudaEventCreate(&e));
        cudaGraph_t g;
        MT_CUDA(cudaStreamBeginCapture(S->s, cudaStreamCaptureModeThreadLocal));
        for (int64_t k = 0; k < nsteps; ++k)
            g_timed->per_step = solid_step_any(S, CTRL_STEP, &g_timed->ev[(size_t)k * 6]);
        MT_CUDA(cudaStreamEndCapture(S->s, &g));
        MT_CUDA(cudaGraphInstantiate(&g_timed->exec, g, 0));
        cudaGraphDestroy(g);
    }
    if (S->d == 2) solid_init_dt<2>(S); else solid_init_dt<3>(S);
    MT_CUDA(cudaGraphLaunch(g_timed->exec, S->s));
    S->launches += nsteps * g_timed->per_step;
    S->pull_ctrl();
    check_solid_errors(S);
    for (int k = 0; k < 7; ++k) timing[k] = 0.0;
    float ms = 0.f;
    MT_CUDA(cudaEventElapsedTime(&ms, g_timed->ev[0], g_timed->ev[(size_t)nsteps * 6 - 1]));
    timing[0] = ms;
    for (int64_t k = 0; k < nsteps; ++k)
        for (int q = 0; q < 5; ++q) {
            MT_CUDA(cudaEventElapsedTime(&ms, g_timed->ev[(size_t)k * 6 + q], g_timed->ev[(size_t)k * 6 + q + 1]));
            timing[1 + q] += ms;
        }
    timing[6] = (double)(nsteps * g_timed->per_step);
    API_END
}

// ------------------------------------------------------------- multi-rank phases

// field 0: velocity; field 1: T~ of the divergence record (the receiver
// completes the record with its own copy of the reference position)
template <int D> __global__ void k_pack(int64_t n, int64_t m, const int64_t *__restrict__ ids, const void *V,
                                        const double *__restrict__ T, const double4 *__restrict__ XV, int field,
                                        double *out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int64_t i = ids[k];
    if (field == 0) {
        double v[3];
        vget(reinterpret_cast<const typename VT<D>::T *>(V)[i], v);
#pragma unroll
        for (int c = 0; c < D; ++c) out[k * D + c] = v[c];
    } else {
        double t[D * D], x[3];
        dload<D>(T, n, XV, i, t, x);
#pragma unroll
        for (int c = 0; c < D * D; ++c) out[k * D * D + c] = t[c];
    }
}

template <int D> __global__ void k_unpack(int64_t n, int64_t m, const int64_t *__restrict__ ids, void *V, double *T,
                                          const double4 *__restrict__ XV, int field,
                                          const double *__restrict__ in) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= m) return;
    const int64_t i = ids[k];
    if (field == 0) {
        double v[3] = {0, 0, 0};
#pragma unroll
        for (int c = 0; c < D; ++c) v[c] = in[k * D + c];
        typename VT<D>::T w;
        vset(w, v);
        reinterpret_cast<typename VT<D>::T *>(V)[i] = w;
    } else {
        double t[D * D];
#pragma unroll
        for (int c = 0; c < D * D; ++c) t[c] = in[k * D * D + c];
        dstore_raw<D>(T, n, i, t, XV[i]);
    }
}

extern "C" mtsph_status mtsph_solid_set_step(mtsph_solid *S, double dt, double eta) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_set_step: null handle");
    API_BEGIN
    S->pull_ctrl();
    S->hc->dt = dt;
    S->hc->eta = eta;
    S->hc->done = 0;
    S->hc->err_inv = S->hc->err_rm = ~0ull;
    S->hc->remote_err = 0;
    S->push_ctrl();
    API_END
}

extern "C" mtsph_status mtsph_solid_colours(const mtsph_solid *S, int *nc) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_colours: null handle");
    *nc = S->nb.sweep == 3 ? (int)S->tiled.colour_ptr.size() - 1 : 0;
    return MTSPH_OK;
}

template <int D> static void solid_phase(mtsph_solid *S, int phase, int arg, double out[2]) {
    SolidArgs A = S->args();
    const unsigned nb = blocks_for(S->n);
    cudaStream_t s = S->s;
    out[0] = out[1] = 0.0;
    switch (phase) {
    case MTSPH_PHASE_KICK_DRIFT:
        k_solid_kick_drift<D><<<nb, 256, 0, s>>>(A);
        S->launches += 1;
        break;
    case MTSPH_PHASE_STRESS:
        S->launches += launch_stress_gather<D>(S, A, s);
        launch_rmap<D>(S, A, s);
        S->launches += 1;
        break;
    case MTSPH_PHASE_ACCEL: {
        S->part.zero(s);
        S->launches += launch_accel_gather<D>(S, A, s);
        MT_LAUNCH_CHECK();
        std::vector<double> h((size_t)2 * S->nblk);
        S->part.download(h.data(), h.size(), s);
        MT_CUDA(cudaStreamSynchronize(s));
        for (int b = 0; b < S->nblk; ++b) {
            out[0] += h[b];
            out[1] = std::max(out[1], h[S->nblk + b]);
        }
        break;
    }
    case MTSPH_PHASE_SWEEP: {
        if (S->nb.sweep != 3) throw Error(MTSPH_ERR_ARG, "sweep phases need the tiled schedule");
        const int c = arg & 63, dir = arg >= 64 ? -1 : 1;
        const TiledSched &t = S->tiled;
        if (c + 1 >= (int)t.colour_ptr.size()) throw Error(MTSPH_ERR_ARG, "colour out of range");
        const int64_t t0 = t.colour_ptr[c], t1 = t.colour_ptr[c + 1];
        if (t1 > t0) {
            k_sweep_tiled<D><<<(unsigned)(t1 - t0), t.threads, tiled_smem_bytes(t, D), s>>>(S->tiled_args(), t0, dir,
                                                                                           S->ctrl.p);
            S->launches += 1;
        }
        break;
    }
    case MTSPH_PHASE_VMAX:
    case MTSPH_PHASE_AMAX: {
        const int with_a = phase == MTSPH_PHASE_AMAX ? 1 : 0;
        S->part.zero(s);
        k_solid_vmax<D><<<nb, 256, 0, s>>>(A, with_a);
        MT_LAUNCH_CHECK();
        S->launches += 1;
        std::vector<double> h((size_t)3 * S->nblk);
        S->part.download(h.data(), h.size(), s);
        MT_CUDA(cudaStreamSynchronize(s));
        for (int b = 0; b < S->nblk; ++b) {
            out[0] = std::max(out[0], h[2 * S->nblk + b]);
            out[1] = std::max(out[1], h[S->nblk + b]);
        }
        break;
    }
    default:
        throw Error(MTSPH_ERR_ARG, "unknown phase");
    }
    MT_LAUNCH_CHECK();
    MT_CUDA(cudaStreamSynchronize(s));
}

extern "C" mtsph_status mtsph_solid_phase(mtsph_solid *S, int phase, int arg, double out[2]) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_phase: null handle");
    API_BEGIN
    if (S->prec != 64) throw Error(MTSPH_ERR_ARG, "multi-rank phases run in fp64");
    if (S->d == 2) solid_phase<2>(S, phase, arg, out); else solid_phase<3>(S, phase, arg, out);
    if (phase == MTSPH_PHASE_STRESS) {
        S->pull_ctrl();
        check_solid_errors(S);
    }
    API_END
}

// ---- device-controlled multi-rank loop: the phases are only enqueued on
// the solid's stream (no host synchronisation), the rank reductions go
// through a device buffer the caller all-gathers (NCCL), and the control
// kernel applies the stopping rule on the device of every rank.

template <int D> static void solid_phase_async(mtsph_solid *S, int phase, int arg) {
    SolidArgs A = S->args();
    const unsigned nb = blocks_for(S->n);
    cudaStream_t s = S->s;
    switch (phase) {
    case MTSPH_PHASE_KICK_DRIFT:
        k_solid_kick_drift<D><<<nb, 256, 0, s>>>(A);
        S->launches += 1;
        break;
    case MTSPH_PHASE_STRESS:
        S->launches += launch_stress_gather<D>(S, A, s);
        launch_rmap<D>(S, A, s);
        S->launches += 1;
        break;
    case MTSPH_PHASE_ACCEL:
        S->launches += launch_accel_gather<D>(S, A, s);
        break;
    case MTSPH_PHASE_SWEEP: {
        if (S->nb.sweep != 3) throw Error(MTSPH_ERR_ARG, "sweep phases need the tiled schedule");
        const int c = arg & 63, dir = arg >= 64 ? -1 : 1;
        const TiledSched &t = S->tiled;
        if (c + 1 >= (int)t.colour_ptr.size()) throw Error(MTSPH_ERR_ARG, "colour out of range");
        const int64_t t0 = t.colour_ptr[c], t1 = t.colour_ptr[c + 1];
        if (t1 > t0) {
            k_sweep_tiled<D><<<(unsigned)(t1 - t0), t.threads, tiled_smem_bytes(t, D), s>>>(S->tiled_args(), t0, dir,
                                                                                           S->ctrl.p);
            S->launches += 1;
        }
        break;
    }
    case MTSPH_PHASE_VMAX:
    case MTSPH_PHASE_AMAX:
        k_solid_vmax<D><<<nb, 256, 0, s>>>(A, phase == MTSPH_PHASE_AMAX ? 1 : 0);
        S->launches += 1;
        break;
    case MTSPH_PHASE_SWEEP_ALL:
        if (S->nb.sweep != 3) throw Error(MTSPH_ERR_ARG, "sweep phases need the tiled schedule");
        if (!S->nb.ghost_internal.empty())
            for (uint8_t g : S->nb.ghost_internal)
                if (g) throw Error(MTSPH_ERR_ARG, "the one-launch sweep needs a rank without ghosts");
        S->launches += launch_tiled_sweep<D>(S->tiled, S->tiled_args(), S->ctrl.p, s);
        break;
    default:
        throw Error(MTSPH_ERR_ARG, "unknown phase");
    }
    MT_LAUNCH_CHECK();
}

extern "C" mtsph_status mtsph_solid_phase_async(mtsph_solid *S, int phase, int arg) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_phase_async: null handle");
    API_BEGIN
    if (S->prec != 64) throw Error(MTSPH_ERR_ARG, "multi-rank phases run in fp64");
    if (S->d == 2) solid_phase_async<2>(S, phase, arg); else solid_phase_async<3>(S, phase, arg);
    API_END
}

extern "C" mtsph_status mtsph_solid_begin_loop(mtsph_solid *S, const mtsph_inner_params *p) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_begin_loop: null handle");
    API_BEGIN
    S->pull_ctrl();
    Ctrl *c = S->hc;
    c->eta = p->eta;
    c->cfl = p->cfl;
    c->criterion = p->criterion;
    c->dt_outer = p->dt_outer;
    c->max_inner = p->max_inner;
    c->min_inner = p->min_inner < 1 ? 1 : p->min_inner;
    c->n_inner = 0;
    c->done = 0;
    c->cap_hit = 0;
    c->min_dt = INFINITY;
    c->err_inv = c->err_rm = ~0ull;
    c->remote_err = 0;
    S->push_ctrl();
    API_END
}

extern "C" mtsph_status mtsph_solid_rank_partials(mtsph_solid *S, int mode, double *dev_out) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_rank_partials: null handle");
    API_BEGIN
    if (mode != CTRL_INIT && mode != CTRL_STEP) throw Error(MTSPH_ERR_ARG, "mode: 0 (initial step) or 1 (step)");
    k_rank_partials<<<1, 256, 0, S->s>>>(S->ctrl.p, S->part.p, S->nblk, mode, dev_out);
    MT_LAUNCH_CHECK();
    S->launches += 1;
    API_END
}

extern "C" mtsph_status mtsph_solid_control_ranks(mtsph_solid *S, const double *dev_gathered, int nranks,
                                                  int mode) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_control_ranks: null handle");
    API_BEGIN
    if (mode != CTRL_INIT && mode != CTRL_STEP) throw Error(MTSPH_ERR_ARG, "mode: 0 (initial step) or 1 (step)");
    if (nranks < 1) throw Error(MTSPH_ERR_ARG, "nranks must be positive");
    k_ctrl_ranks<<<1, 32, 0, S->s>>>(S->ctrl.p, dev_gathered, nranks, mode);
    MT_LAUNCH_CHECK();
    S->launches += 1;
    API_END
}

extern "C" mtsph_status mtsph_solid_loop_state(mtsph_solid *S, mtsph_inner_result *r, int *done) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_loop_state: null handle");
    API_BEGIN
    S->pull_ctrl();
    const Ctrl *c = S->hc;
    *done = c->done;
    r->n_inner = c->n_inner;
    r->cap_hit = c->cap_hit;
    r->ek = c->ek;
    r->min_dt = c->min_dt;
    r->last_dt = c->last_dt;
    check_solid_errors(S);
    API_END
}

static void pack_common(mtsph_solid *S, const char *field, int64_t m, const int64_t *ids, double *host,
                        const double *in, bool pack) {
    if (S->prec != 64) throw Error(MTSPH_ERR_ARG, "multi-rank exchanges run in fp64");
    const std::string f(field);
    const int which = f == "vel" ? 0 : (f == "T" ? 1 : -1);
    if (which < 0) throw Error(MTSPH_ERR_ARG, "pack fields are 'vel' and 'T'");
    if (m <= 0) return;
    if (S->iperm_h.empty()) {
        S->iperm_h.resize(S->n);
        S->nb.iperm.download(S->iperm_h.data(), S->n, S->s);
        MT_CUDA(cudaStreamSynchronize(S->s));
    }
    std::vector<int64_t> internal(m);
    for (int64_t k = 0; k < m; ++k) {
        if (ids[k] < 0 || ids[k] >= S->n) throw Error(MTSPH_ERR_ARG, "particle id out of range");
        internal[k] = S->iperm_h[ids[k]];
    }
    const int w = which == 0 ? S->d : S->d * S->d;
    DBuf<int64_t> dids(m);
    DBuf<double> buf((size_t)m * w);
    dids.upload(internal.data(), m, S->s);
    if (pack) {
        if (S->d == 2)
            k_pack<2><<<blocks_for(m), 256, 0, S->s>>>(S->n, m, dids.p, S->V.p, S->T.p, S->nb.XV.p, which, buf.p);
        else
            k_pack<3><<<blocks_for(m), 256, 0, S->s>>>(S->n, m, dids.p, S->V.p, S->T.p, S->nb.XV.p, which, buf.p);
        MT_LAUNCH_CHECK();
        buf.download(host, (size_t)m * w, S->s);
    } else {
        buf.upload(in, (size_t)m * w, S->s);
        if (S->d == 2)
            k_unpack<2><<<blocks_for(m), 256, 0, S->s>>>(S->n, m, dids.p, S->V.p, S->T.p, S->nb.XV.p, which, buf.p);
        else
            k_unpack<3><<<blocks_for(m), 256, 0, S->s>>>(S->n, m, dids.p, S->V.p, S->T.p, S->nb.XV.p, which, buf.p);
        MT_LAUNCH_CHECK();
    }
    S->launches += 1;
    MT_CUDA(cudaStreamSynchronize(S->s));
}

extern "C" mtsph_status mtsph_solid_pack(mtsph_solid *S, const char *field, int64_t m, const int64_t *ids,
                                         double *host) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_pack: null handle");
    API_BEGIN
    pack_common(S, field, m, ids, host, nullptr, true);
    API_END
}

extern "C" mtsph_status mtsph_solid_unpack(mtsph_solid *S, const char *field, int64_t m, const int64_t *ids,
                                           const double *host) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_unpack: null handle");
    API_BEGIN
    pack_common(S, field, m, ids, nullptr, host, false);
    API_END
}

// ---- device-resident exchange

static int pack_field(const char *field) {
    const std::string f(field ? field : "");
    const int which = f == "vel" ? 0 : (f == "T" ? 1 : -1);
    if (which < 0) throw Error(MTSPH_ERR_ARG, "pack fields are 'vel' and 'T'");
    return which;
}

extern "C" mtsph_status mtsph_solid_internal_ids(mtsph_solid *S, int64_t m, const int64_t *ids,
                                                 int64_t *internal) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_internal_ids: null handle");
    API_BEGIN
    if (S->iperm_h.empty()) {
        S->iperm_h.resize(S->n);
        S->nb.iperm.download(S->iperm_h.data(), S->n, S->s);
        MT_CUDA(cudaStreamSynchronize(S->s));
    }
    for (int64_t k = 0; k < m; ++k) {
        if (ids[k] < 0 || ids[k] >= S->n) throw Error(MTSPH_ERR_ARG, "particle id out of range");
        internal[k] = S->iperm_h[ids[k]];
    }
    API_END
}

extern "C" mtsph_status mtsph_solid_stream(const mtsph_solid *S, void **stream) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_stream: null handle");
    *stream = (void *)S->s;
    return MTSPH_OK;
}

extern "C" mtsph_status mtsph_solid_pack_device(mtsph_solid *S, const char *field, int64_t m,
                                                const int64_t *ids, double *out) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_pack_device: null handle");
    API_BEGIN
    if (S->prec != 64) throw Error(MTSPH_ERR_ARG, "multi-rank exchanges run in fp64");
    const int which = pack_field(field);
    if (m <= 0) return MTSPH_OK;
    if (S->d == 2) k_pack<2><<<blocks_for(m), 256, 0, S->s>>>(S->n, m, ids, S->V.p, S->T.p, S->nb.XV.p, which, out);
    else k_pack<3><<<blocks_for(m), 256, 0, S->s>>>(S->n, m, ids, S->V.p, S->T.p, S->nb.XV.p, which, out);
    MT_LAUNCH_CHECK();
    S->launches += 1;
    API_END
}

extern "C" mtsph_status mtsph_solid_unpack_device(mtsph_solid *S, const char *field, int64_t m,
                                                  const int64_t *ids, const double *in) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_unpack_device: null handle");
    API_BEGIN
    if (S->prec != 64) throw Error(MTSPH_ERR_ARG, "multi-rank exchanges run in fp64");
    const int which = pack_field(field);
    if (m <= 0) return MTSPH_OK;
    if (S->d == 2) k_unpack<2><<<blocks_for(m), 256, 0, S->s>>>(S->n, m, ids, S->V.p, S->T.p, S->nb.XV.p, which, in);
    else k_unpack<3><<<blocks_for(m), 256, 0, S->s>>>(S->n, m, ids, S->V.p, S->T.p, S->nb.XV.p, which, in);
    MT_LAUNCH_CHECK();
    S->launches += 1;
    API_END
}

extern "C" mtsph_status mtsph_solid_measure(mtsph_solid *S, double out[5]) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_measure: null handle");
    API_BEGIN
    sync64(S);
    SolidArgs A = S->args();
    const int nb = S->nblk;
    if (S->d == 2) k_solid_measure<2><<<nb, 256, 0, S->s>>>(A, S->meas.p);
    else k_solid_measure<3><<<nb, 256, 0, S->s>>>(A, S->meas.p);
    MT_LAUNCH_CHECK();
    S->launches += 1;
    std::vector<double> h((size_t)5 * nb);
    S->meas.download(h.data(), h.size(), S->s);
    MT_CUDA(cudaStreamSynchronize(S->s));
    double fx = 0.0, rad = 0.0, amax = 0.0, amin = 1e308, bad = 0.0;
    for (int b = 0; b < nb; ++b) {
        fx += h[b];
        rad = std::max(rad, h[nb + b]);
        amax = std::max(amax, h[2 * nb + b]);
        amin = std::min(amin, h[3 * nb + b]);
        bad = std::max(bad, h[4 * nb + b]);
    }
    out[0] = -fx;
    out[1] = rad;
    out[2] = S->mat.plastic ? amax : 0.0;
    out[3] = S->mat.plastic && amin < 1e308 ? amin : 0.0;   // no mid-span particles: 0
    out[4] = bad > 0 ? 0.0 : 1.0;
    API_END
}

enum FieldKind { FK_SOA_VEC, FK_SOA_TEN, FK_SCALAR, FK_VEL, FK_REF };

extern "C" mtsph_status mtsph_solid_get(mtsph_solid *S, const char *field, double *host) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_get: null handle");
    API_BEGIN
    sync64(S);
    const int64_t n = S->n;
    const int d = S->d;
    std::vector<int64_t> perm(n);
    S->nb.perm.download(perm.data(), n, S->s);
    std::string f(field);
    std::vector<double> buf;
    auto soa = [&](const DBuf<double> &src, int comps) {
        buf.resize((size_t)comps * n);
        src.download(buf.data(), buf.size(), S->s);
        MT_CUDA(cudaStreamSynchronize(S->s));
        for (int64_t k = 0; k < n; ++k)
            for (int c = 0; c < comps; ++c) host[perm[k] * comps + c] = buf[(size_t)c * n + k];
    };
    if (f == "pos") soa(S->x, d);
    else if (f == "accel") soa(S->a, d);
    else if (f == "F") soa(S->F, d * d);
    else if (f == "cp_inv") soa(S->cp, d * d);
    else if (f == "alpha") soa(S->alpha, 1);
    else if (f == "vel" || f == "ref_pos") {
        const int stride = (f == "ref_pos" || d == 3) ? 4 : 2;
        buf.resize((size_t)stride * n);
        if (f == "vel") MT_CUDA(cudaMemcpyAsync(buf.data(), S->V.p, buf.size() * 8, cudaMemcpyDeviceToHost, S->s));
        else MT_CUDA(cudaMemcpyAsync(buf.data(), S->nb.XV.p, buf.size() * 8, cudaMemcpyDeviceToHost, S->s));
        MT_CUDA(cudaStreamSynchronize(S->s));
        for (int64_t k = 0; k < n; ++k)
            for (int c = 0; c < d; ++c) host[perm[k] * d + c] = buf[(size_t)k * stride + c];
    } else throw Error(MTSPH_ERR_ARG, "unknown solid field " + f);
    API_END
}

extern "C" mtsph_status mtsph_solid_set(mtsph_solid *S, const char *field, const double *host) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_set: null handle");
    API_BEGIN
    sync64(S);
    const int64_t n = S->n;
    const int d = S->d;
    std::vector<int64_t> perm(n);
    S->nb.perm.download(perm.data(), n, S->s);
    MT_CUDA(cudaStreamSynchronize(S->s));
    std::string f(field);
    std::vector<double> buf;
    auto soa = [&](DBuf<double> &dst, int comps) {
        buf.resize((size_t)comps * n);
        for (int64_t k = 0; k < n; ++k)
            for (int c = 0; c < comps; ++c) buf[(size_t)c * n + k] = host[perm[k] * comps + c];
        dst.upload(buf.data(), buf.size(), S->s);
    };
    if (f == "pos") soa(S->x, d);
    else if (f == "accel") soa(S->a, d);
    else if (f == "F") soa(S->F, d * d);
    else if (f == "cp_inv") soa(S->cp, d * d);
    else if (f == "alpha") soa(S->alpha, 1);
    else if (f == "vel") {
        const int stride = d == 3 ? 4 : 2;
        buf.assign((size_t)stride * n, 0.0);
        for (int64_t k = 0; k < n; ++k)
            for (int c = 0; c < d; ++c) buf[(size_t)k * stride + c] = host[perm[k] * d + c];
        MT_CUDA(cudaMemcpyAsync(S->V.p, buf.data(), buf.size() * 8, cudaMemcpyHostToDevice, S->s));
    } else throw Error(MTSPH_ERR_ARG, "unknown or read-only solid field " + f);
    sync32(S);
    MT_CUDA(cudaStreamSynchronize(S->s));
    API_END
}

extern "C" mtsph_status mtsph_solid_sizes(const mtsph_solid *S, int64_t out[4]) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_sizes: null handle");
    const NbhDev &nb = S->nb;
    out[0] = nb.nnz;
    out[1] = nb.sweep == 3 ? S->tiled.npairs : nb.npairs;
    out[2] = nb.sweep == 3 ? S->tiled.npairs : nb.ngroups;
    int64_t ph = 0;
    if (nb.sweep == 3)
        for (size_t k = 0; k + 1 < S->tiled.colour_ptr.size(); ++k) ph += S->tiled.colour_ptr[k + 1] > S->tiled.colour_ptr[k];
    if (nb.sweep == 1) ph = nb.nlevels;
    else if (nb.sweep == 2)
        for (size_t k = 0; k + 1 < nb.colour_task_ptr.size(); ++k) ph += nb.colour_task_ptr[k + 1] > nb.colour_task_ptr[k];
    out[3] = ph;
    return MTSPH_OK;
}

extern "C" mtsph_status mtsph_solid_launches(const mtsph_solid *S, int64_t *count) {
    if (!S) return fail(MTSPH_ERR_ARG, "mtsph_solid_launches: null handle");
    *count = S->launches;
    return MTSPH_OK;
}

#include "porous_api.cuh"
#include "layer1_api.cuh"
