// common.cuh -- shared device helpers for the mtsph B200 kernels.
//
// Everything here is header-only and compiled into one translation unit
// (mtsph_b200.cu).  fp64 throughout: the reference state is fp64 and the
// parity bar is 1e-10 relative per step.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <thread>
#include <string>
#include <vector>

namespace mtsph {

// ---------------------------------------------------------------- errors

struct Error : std::runtime_error {
    int code;
    std::vector<int64_t> ids;
    Error(int c, const std::string &m, std::vector<int64_t> i = {})
        : std::runtime_error(m), code(c), ids(std::move(i)) {}
};

#define MT_CUDA(expr)                                                          \
    do {                                                                       \
        cudaError_t _e = (expr);                                               \
        if (_e != cudaSuccess)                                                 \
            throw ::mtsph::Error(2, std::string(#expr) + ": " +                \
                                        cudaGetErrorString(_e));               \
    } while (0)

#define MT_LAUNCH_CHECK() MT_CUDA(cudaGetLastError())

constexpr int kThreads = 256;
inline unsigned blocks_for(int64_t n, int t = kThreads) {
    int64_t b = (n + t - 1) / t;
    return (unsigned)(b < 1 ? 1 : b);
}

// MTSPH_VERBOSE=1: wall time since the previous mark, per setup phase, on
// stderr (synchronises the stream; a no-op otherwise)
inline void setup_mark(cudaStream_t s, const char *what) {
    static const bool on = [] { const char *e = std::getenv("MTSPH_VERBOSE"); return e && e[0] == '1'; }();
    if (!on) return;
    static thread_local std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[mtsph] %-24s %8.3f s\n", what, std::chrono::duration<double>(now - last).count());
    last = now;
}

// opt a kernel into the largest dynamic shared memory the device offers
// (the opt-in limit covers static + dynamic)
inline void allow_max_dynamic_smem(const void *fn) {
    int dev = 0, optin = 0;
    cudaFuncAttributes fa{};
    MT_CUDA(cudaGetDevice(&dev));
    MT_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    MT_CUDA(cudaFuncGetAttributes(&fa, fn));
    MT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 optin - (int)fa.sharedSizeBytes));
}

// memcpy split over host threads (first-touch page faults of a fresh
// multi-GB destination serialise a single-threaded copy at ~2 GB/s)
inline void par_memcpy(void *dst, const void *src, size_t len) {
    constexpr int kThreadsCopy = 8;
    if (len < (size_t(4) << 20)) { std::memcpy(dst, src, len); return; }
    std::thread th[kThreadsCopy];
    const size_t per = (len + kThreadsCopy - 1) / kThreadsCopy;
    for (int k = 0; k < kThreadsCopy; ++k) {
        const size_t off = k * per, n = off < len ? std::min(per, len - off) : 0;
        th[k] = std::thread([=] { if (n) std::memcpy(static_cast<char *>(dst) + off, static_cast<const char *>(src) + off, n); });
    }
    for (auto &t : th) t.join();
}

// Large host<->device copies of pageable host memory through a
// double-buffered pinned staging ring (a plain pageable cudaMemcpy ran at
// ~3 GB/s for the multi-GB setup arrays): the DMA of one chunk overlaps the
// host memcpy of the other.  Synchronous on return.
inline void copy_staged(void *dst, const void *src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    constexpr size_t kChunk = size_t(64) << 20;
    if (bytes < (size_t(8) << 20)) {  // small: not worth the staging
        MT_CUDA(cudaMemcpyAsync(dst, src, bytes, kind, s));
        MT_CUDA(cudaStreamSynchronize(s));
        return;
    }
    static std::mutex mu;
    std::lock_guard<std::mutex> lock(mu);
    static char *stage[2] = {nullptr, nullptr};
    static cudaEvent_t done[2];
    if (!stage[0])
        for (int k = 0; k < 2; ++k) {
            MT_CUDA(cudaMallocHost(&stage[k], kChunk));
            MT_CUDA(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
        }
    const size_t nchunk = (bytes + kChunk - 1) / kChunk;
    char *d = static_cast<char *>(dst);
    const char *h = static_cast<const char *>(src);
    if (kind == cudaMemcpyHostToDevice) {
        for (size_t c = 0; c < nchunk; ++c) {
            const int k = (int)(c & 1);
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            if (c >= 2) MT_CUDA(cudaEventSynchronize(done[k]));  // buffer k free again
            par_memcpy(stage[k], h + off, len);
            MT_CUDA(cudaMemcpyAsync(d + off, stage[k], len, kind, s));
            MT_CUDA(cudaEventRecord(done[k], s));
        }
    } else {
        // D2H: chunk c+1's DMA runs while chunk c is copied out
        auto issue = [&](size_t c) {
            const int k = (int)(c & 1);
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            MT_CUDA(cudaMemcpyAsync(stage[k], h + off, len, kind, s));
            MT_CUDA(cudaEventRecord(done[k], s));
        };
        issue(0);
        for (size_t c = 0; c < nchunk; ++c) {
            if (c + 1 < nchunk) issue(c + 1);
            const int k = (int)(c & 1);
            const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
            MT_CUDA(cudaEventSynchronize(done[k]));
            par_memcpy(d + off, stage[k], len);
        }
    }
    MT_CUDA(cudaStreamSynchronize(s));
}

// device buffer with RAII
template <class T> struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t cnt) { alloc(cnt); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t cnt) {
        release();
        n = cnt;
        if (cnt) MT_CUDA(cudaMalloc(&p, cnt * sizeof(T)));
    }
    void zero(cudaStream_t s = 0) {
        if (n) MT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    // small copies stay asynchronous; >= 8 MB go through the pinned staging
    // ring (synchronous) -- setup-time arrays of pageable host memory
    void upload(const T *h, size_t cnt, cudaStream_t s = 0) {
        if (cnt > n) alloc(cnt);
        if (cnt * sizeof(T) >= (size_t(8) << 20)) copy_staged(p, h, cnt * sizeof(T), cudaMemcpyHostToDevice, s);
        else if (cnt) MT_CUDA(cudaMemcpyAsync(p, h, cnt * sizeof(T), cudaMemcpyHostToDevice, s));
    }
    void download(T *h, size_t cnt, cudaStream_t s = 0) const {
        if (cnt * sizeof(T) >= (size_t(8) << 20)) copy_staged(h, p, cnt * sizeof(T), cudaMemcpyDeviceToHost, s);
        else if (cnt) MT_CUDA(cudaMemcpyAsync(h, p, cnt * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    T *get() const { return p; }
};

// ---------------------------------------------------------------- kernel

// Anisotropic Wendland C2 kernel, support 2h (kernels.py:76-118).  Scaled
// separation u_k = r_k / h_k, q = |u|:
//   w(q) = (1 - q/2)^4 (1 + 2q),  dw/dq = -5 q (1 - q/2)^3
//   grad_k = pref * dw/dq / q * u_k / h_k = pref * (-5 (1-q/2)^3) u_k / h_k
struct KSpec {
    double h[3];
    double inv_h[3];
    double pref;   // sigma_d / prod(h)
    double h_min;
    double inv_h2[3];  // 1 / h_k^2
    double pref5;      // -5 pref
};

// Evaluated as w_k = r_k / h_k^2, q^2 = sum r_k w_k, grad_k = -5 pref
// (1-q/2)^3 w_k: the same value as the form above up to rounding, with
// fewer FP64 operations in the neighbour loops (9 instead of 13 besides
// the square root).
// magnitude factor and scaled separation: gradW = mag * w
template <int D>
__device__ __forceinline__ double grad_mag(const double *rel, const KSpec &ks, double *w) {
    double q2 = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) { w[k] = rel[k] * ks.inv_h2[k]; q2 = fma(rel[k], w[k], q2); }
    const double q = sqrt(q2);
    const double t = 1.0 - 0.5 * q;
    return (q < 2.0) ? ks.pref5 * (t * t * t) : 0.0;
}
template <int D>
__device__ __forceinline__ void grad_w(const double *rel, const KSpec &ks, double *g) {
    double w[D];
    const double mag = grad_mag<D>(rel, ks, w);
#pragma unroll
    for (int k = 0; k < D; ++k) g[k] = mag * w[k];
}
// gradW from a stored magnitude factor (gather_csr.cuh build_chunked): the
// same products as grad_w, without the square root and the polynomial
template <int D>
__device__ __forceinline__ void grad_w_mag(const double *rel, const KSpec &ks, double mag, double *g) {
#pragma unroll
    for (int k = 0; k < D; ++k) g[k] = mag * (rel[k] * ks.inv_h2[k]);
}

// 32 B accesses.  sm_100 has 256-bit global loads/stores (SASS
// LDG.E.ENL2.256 / STG.E.ENL2.256) but nvcc splits a plain double4 access
// into two 128-bit ones, each of which costs the L1 a tag lookup on the same
// sector.  In the neighbour gathers that doubled the sectors per request, so
// the gathered records go through these explicit v4.f64 forms.
//   ldg4: read-only for the whole kernel (non-coherent path)
//   ld4 / st4: coherent, for records the kernel also writes
__device__ __forceinline__ double4 ldg4(const double4 *p) {
    double4 r;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
    return r;
}
// L2-coherent 32 B load (bypasses L1): data another SM wrote during this launch
__device__ __forceinline__ double4 ldcg4(const double4 *p) {
    double4 r;
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ double4 ld4(const double4 *p) {
    double4 r;
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p) : "memory");
    return r;
}
__device__ __forceinline__ void st4(double4 *p, const double4 &v) {
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                 : "memory");
}

// ------------------------------------------------------ small tensors

template <int D> __device__ __forceinline__ double det_d(const double *t) {
    if (D == 1) return t[0];
    if (D == 2) return t[0] * t[3] - t[1] * t[2];
    return t[0] * (t[4] * t[8] - t[5] * t[7]) - t[1] * (t[3] * t[8] - t[5] * t[6]) +
           t[2] * (t[3] * t[7] - t[4] * t[6]);
}

// adjugate / det, reference tensors.py:170 layout
template <int D> __device__ __forceinline__ void inv_d(const double *t, double j, double *o) {
    if (D == 1) { o[0] = 1.0 / j; return; }
    if (D == 2) {
        o[0] = t[3] / j; o[1] = -t[1] / j; o[2] = -t[2] / j; o[3] = t[0] / j;
        return;
    }
    o[0] = (t[4] * t[8] - t[5] * t[7]) / j;
    o[1] = (t[2] * t[7] - t[1] * t[8]) / j;
    o[2] = (t[1] * t[5] - t[2] * t[4]) / j;
    o[3] = (t[5] * t[6] - t[3] * t[8]) / j;
    o[4] = (t[0] * t[8] - t[2] * t[6]) / j;
    o[5] = (t[2] * t[3] - t[0] * t[5]) / j;
    o[6] = (t[3] * t[7] - t[4] * t[6]) / j;
    o[7] = (t[1] * t[6] - t[0] * t[7]) / j;
    o[8] = (t[0] * t[4] - t[1] * t[3]) / j;
}

template <int D> __device__ __forceinline__ void mm(const double *a, const double *b, double *o) {
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s += a[r * D + k] * b[k * D + c];
            o[r * D + c] = s;
        }
}

// a @ b^T
template <int D> __device__ __forceinline__ void mmt(const double *a, const double *b, double *o) {
#pragma unroll
    for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s += a[r * D + k] * b[c * D + k];
            o[r * D + c] = s;
        }
}

// det^(-1/d) without pow for d = 2, 3
template <int D> __device__ __forceinline__ double det_pow_minus_inv_d(double j) {
    if (D == 1) return 1.0 / j;
    if (D == 2) return rsqrt(j);
    return rcbrt(j);
}

// --------------------------------------------------- reductions (fixed order)

// block-level sum/max with a fixed tree shape: deterministic for a fixed
// launch configuration.
template <int BT> __device__ __forceinline__ double block_sum(double v, double *sh) {
    const int t = threadIdx.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((t & 31) == 0) sh[t >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (t < 32) {
        r = (t < BT / 32) ? sh[t] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r += __shfl_down_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

// (the lanes past the block's warp count pad with -inf / +inf, so any sign
// of value reduces correctly)
template <int BT> __device__ __forceinline__ double block_max(double v, double *sh) {
    const int t = threadIdx.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    if ((t & 31) == 0) sh[t >> 5] = v;
    __syncthreads();
    double r = -INFINITY;
    if (t < 32) {
        r = (t < BT / 32) ? sh[t] : -INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_down_sync(0xffffffffu, r, o));
    }
    __syncthreads();
    return r;
}
template <int BT> __device__ __forceinline__ double block_min(double v, double *sh) {
    const int t = threadIdx.x;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
    if ((t & 31) == 0) sh[t >> 5] = v;
    __syncthreads();
    double r = INFINITY;
    if (t < 32) {
        r = (t < BT / 32) ? sh[t] : INFINITY;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r = fmin(r, __shfl_down_sync(0xffffffffu, r, o));
    }
    __syncthreads();
    return r;
}

// ordered uint64 key of a double (for radix sorts that mimic np.lexsort);
// +0.0 and -0.0 map to the same key, as numpy compares them equal.
__device__ __forceinline__ uint64_t dkey(double x) {
    uint64_t b = (uint64_t)__double_as_longlong(x);
    if ((b << 1) == 0) b = 0;  // -0.0 -> +0.0
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__host__ __device__ __forceinline__ uint64_t spread3(uint64_t v) {  // 21 bits -> every 3rd
    v &= 0x1fffffull;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}
__host__ __device__ __forceinline__ uint64_t spread2(uint64_t v) {  // 32 bits -> every 2nd
    v &= 0xffffffffull;
    v = (v | v << 16) & 0x0000ffff0000ffffull;
    v = (v | v << 8) & 0x00ff00ff00ff00ffull;
    v = (v | v << 4) & 0x0f0f0f0f0f0f0f0full;
    v = (v | v << 2) & 0x3333333333333333ull;
    v = (v | v << 1) & 0x5555555555555555ull;
    return v;
}

}  // namespace mtsph
