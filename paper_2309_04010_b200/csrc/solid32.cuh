// solid32.cuh -- fp32 variant of the inner relaxation step.
//
// The north star asks for fp64 state (the reference's, parity-tested) and
// an fp32 variant reported separately.  This is that variant: the same
// step as solid.cuh / gather_csr.cuh / the tiled sweep, with every array
// the step streams in single precision, so each gathered record is half
// the bytes (X|V0 and v: 16 B, the divergence record 48 B) and the sweep's
// shared-memory halo is one float4 per particle.
//
// Stored as deviations so single precision keeps the increments of a
// relaxation step (dt * L ~ 1e-7 next to 1 would round away):
//   u  = x - X        (displacement, not the current position)
//   H  = F - I        (displacement gradient)
//   Hc = C_p^-1 - I
// The return map (plasticity.py:118) is evaluated in fp64 from these (its
// Newton tolerance, 1e-8 s0, is below fp32 resolution); neighbour sums,
// kernel gradients, the kick/drift and the damping pair updates are fp32.
// Reductions (E_k, |a|max, |v|max) accumulate in fp64 and the control
// kernel (k_ctrl) is the fp64 one, so the stopping rule is unchanged.
//
// The fp64 arrays of mtsph_solid stay allocated as the host-facing mirror:
// mtsph_solid_set_precision converts between the two, get/set/measure go
// through the fp64 copy.
#pragma once

#include "gather_csr.cuh"
#include "tiled.cuh"

namespace mtsph {

struct KSpec32 {
    float inv_h2[3];
    float pref5;   // -5 pref
};

inline KSpec32 kspec32(const KSpec &k) {
    KSpec32 r;
    for (int q = 0; q < 3; ++q) r.inv_h2[q] = (float)k.inv_h2[q];
    r.pref5 = (float)k.pref5;
    return r;
}

// grad_w (common.cuh) in fp32
template <int D>
__device__ __forceinline__ void grad_w32(const float *rel, const KSpec32 &ks, float *g) {
    float w[D];
    float q2 = 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) { w[k] = rel[k] * ks.inv_h2[k]; q2 = fmaf(rel[k], w[k], q2); }
    const float q = sqrtf(q2);
    const float t = 1.f - 0.5f * q;
    const float mag = (q < 2.f) ? ks.pref5 * (t * t * t) : 0.f;
#pragma unroll
    for (int k = 0; k < D; ++k) g[k] = mag * w[k];
}

struct Solid32Args {
    int64_t n;
    const float4 *XV;        // X, V0 (16 B)
    void *V;                 // float2 (2D) / float4 (3D)
    float *u, *a, *H, *Hc, *alpha, *T;   // T: divergence records (DS<D>::n floats)
    const float *B, *G, *mass, *rho0;
    const uint8_t *flags;
    const int64_t *indptr;
    const int32_t *csr;
    const int64_t *cptr;     // chunked index table (gather_csr.cuh), or null
    const int32_t *csr16;
    const int64_t *perm;
    double *part;            // [3][nblk]: ek, amax2, vmax2 (fp64 partials)
    int nblk;
    Ctrl *ctrl;
    KSpec32 ks;
    Mat mat;
};

template <int D> __device__ __forceinline__ void xget32(const float4 &xv, float *x) {
    x[0] = xv.x; x[1] = xv.y;
    if (D == 3) x[2] = xv.z;
}
template <int D> __device__ __forceinline__ float volof32(const float4 &xv) { return D == 3 ? xv.w : xv.z; }

// two floats packed in a double's bit pattern (256-bit records are moved
// with the v4.f64 loads/stores of common.cuh)
__device__ __forceinline__ void unpack2f(double d, float &lo, float &hi) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(d);
    lo = __uint_as_float((unsigned)(u & 0xffffffffull));
    hi = __uint_as_float((unsigned)(u >> 32));
}
__device__ __forceinline__ double pack2f(float lo, float hi) {
    return __longlong_as_double((long long)(((unsigned long long)__float_as_uint(hi) << 32) |
                                            __float_as_uint(lo)));
}

// divergence record, fp32: 3D one 32 B plane (T~00 .. T~21, one 256-bit
// load) and one 16 B plane (X0 X1 X2 T~22) -- two loads per neighbour
// instead of three 16 B ones (accel 3.24 -> 3.12 ms at 10M); 2D
// (T~00 T~01 T~10 T~11), X from XV.  (Interleaving X|V0 with v in one
// 32 B record for the deformation-rate gather was slower: 3.62 -> 3.89 ms.)
template <int D>
__device__ __forceinline__ void dstore32(float *Tp, int64_t n, int64_t a, const float *tt, const float4 &xv) {
    if (D == 3) {
        st4(reinterpret_cast<double4 *>(Tp) + a,
            make_double4(pack2f(tt[0], tt[1]), pack2f(tt[2], tt[3]), pack2f(tt[4], tt[5]), pack2f(tt[6], tt[7])));
        reinterpret_cast<float4 *>(Tp + 8 * n)[a] = make_float4(xv.x, xv.y, xv.z, tt[8]);
    } else {
        reinterpret_cast<float4 *>(Tp)[a] = make_float4(tt[0], tt[1], tt[2], tt[3]);
    }
}
template <int D>
__device__ __forceinline__ void dload32(const float *Tp, int64_t n, const float4 *XV, int64_t b, float *tt,
                                        float *x) {
    if (D == 2) {
        const float4 q0 = __ldg(reinterpret_cast<const float4 *>(Tp) + b);
        tt[0] = q0.x; tt[1] = q0.y; tt[2] = q0.z; tt[3] = q0.w;
        const float4 xv = __ldg(XV + b);
        x[0] = xv.x; x[1] = xv.y;
    } else {
        const double4 q = ldg4(reinterpret_cast<const double4 *>(Tp) + b);
        unpack2f(q.x, tt[0], tt[1]);
        unpack2f(q.y, tt[2], tt[3]);
        unpack2f(q.z, tt[4], tt[5]);
        unpack2f(q.w, tt[6], tt[7]);
        const float4 q2 = __ldg(reinterpret_cast<const float4 *>(Tp + 8 * n) + b);
        tt[8] = q2.w;
        x[0] = q2.x; x[1] = q2.y; x[2] = q2.z;
    }
}

template <int G, int K> __device__ __forceinline__ void group_sum32(float (&v)[K]) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
        for (int k = 0; k < K; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
}

// k_solid_kick_drift in fp32 (u += dt v instead of x += dt v)
template <int D>
__global__ void __launch_bounds__(256) k32_kick_drift(Solid32Args A) {
    using V_t = typename VTR<D, float>::T;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const float dt = (float)c->dt;
    const uint8_t f = A.flags[i];
    V_t *V = reinterpret_cast<V_t *>(A.V);
    float v[3];
    vget(V[i], v);
    if (f & FL_MOVABLE) {
#pragma unroll
        for (int k = 0; k < D; ++k) v[k] += 0.5f * dt * A.a[(int64_t)k * A.n + i];
    }
    if (c->ramp_left > 0) {
        if (f & (FL_LEFT | FL_RIGHT)) {
            const float vbc = (float)(c->ramp_disp / c->dt);
#pragma unroll
            for (int k = 0; k < D; ++k) v[k] = 0.f;
            v[0] = (f & FL_LEFT) ? -vbc : vbc;
        }
    } else if (!(f & FL_MOVABLE)) {
#pragma unroll
        for (int k = 0; k < D; ++k) v[k] = 0.f;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) A.u[(int64_t)k * A.n + i] += dt * v[k];
    V_t w;
    vset(w, v);
    V[i] = w;
}

// k_solid_stress_csr in fp32: H += dt (sum_b V_b (v_b - v_a) (x) gradW) B
template <int D, int G, bool C16 = false>
__global__ void __launch_bounds__(256) k32_stress_csr(Solid32Args A) {
    using V_t = typename VTR<D, float>::T;
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const float dt = (float)c->dt;
    const int64_t n = A.n;
    const int sub = threadIdx.x % G;
    const V_t *V = reinterpret_cast<const V_t *>(A.V);
    for (int it = 0; it < G; ++it) {
        const int64_t i = (int64_t)blockIdx.x * 256 + it * (256 / G) + threadIdx.x / G;
        const bool act = i < n;
        float acc[D * D];
#pragma unroll
        for (int k = 0; k < D * D; ++k) acc[k] = 0.f;
        if (act) {
            float xa[3], va[3];
            xget32<D>(__ldg(A.XV + i), xa);
            vget(vldg(V + i), va);
            auto visit = [&](int32_t b) {
                const float4 xvb = __ldg(A.XV + b);
                float xb[3], vb[3], rel[D], g[D];
                xget32<D>(xvb, xb);
                vget(vldg(V + b), vb);
#pragma unroll
                for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
                grad_w32<D>(rel, A.ks, g);
                const float volb = volof32<D>(xvb);
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    const float dv = volb * (vb[r] - va[r]);
#pragma unroll
                    for (int cc = 0; cc < D; ++cc) acc[r * D + cc] += dv * g[cc];
                }
            };
            if constexpr (C16) {
                walk_chunks<G, false>(A.cptr, A.csr16, i, sub, visit);
            } else {
                const int64_t k1 = A.indptr[i + 1];
                for (int64_t k = A.indptr[i] + sub; k < k1; k += G) visit(__ldg(A.csr + k));
            }
        }
        group_sum32<G>(acc);
        if (act && sub == 0) {
            float Bm[D * D];
#pragma unroll
            for (int k = 0; k < D * D; ++k) Bm[k] = A.B[(int64_t)k * n + i];
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
                for (int cc = 0; cc < D; ++cc) {
                    float l = 0.f;
#pragma unroll
                    for (int k = 0; k < D; ++k) l += acc[r * D + k] * Bm[k * D + cc];
                    A.H[(int64_t)(r * D + cc) * n + i] += dt * l;
                }
        }
    }
}

// k_solid_rmap in fp32 storage: F = I + H, C_p^-1 = I + Hc, the return map
// in fp64, T~ = V0 P B stored in fp32
template <int D, int LAW>
__global__ void __launch_bounds__(256, 2) k32_rmap(Solid32Args A) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= A.n) return;
    Ctrl *c = A.ctrl;
    if (c->done) return;
    const int64_t n = A.n;
    double F[D * D], cp[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) {
        const double id = (k % (D + 1) == 0) ? 1.0 : 0.0;
        F[k] = id + (double)A.H[(int64_t)k * n + i];
        cp[k] = id;
    }
    double alpha = 0.0;
    if (A.mat.plastic) {
#pragma unroll
        for (int k = 0; k < D * D; ++k) cp[k] += (double)A.Hc[(int64_t)k * n + i];
        alpha = (double)A.alpha[i];
    }
    double P[D * D];
    const int rc = return_map_dev<D, LAW>(F, cp, alpha, A.mat, P);
    if (rc) {
        const unsigned long long id = (unsigned long long)A.perm[i];
        if (rc == 1) atomicMin(&c->err_inv, id);
        else atomicMin(&c->err_rm, id);
#pragma unroll
        for (int k = 0; k < D * D; ++k) P[k] = 0.0;
    } else if (A.mat.plastic) {
#pragma unroll
        for (int k = 0; k < D * D; ++k) A.Hc[(int64_t)k * n + i] = (float)(cp[k] - ((k % (D + 1) == 0) ? 1.0 : 0.0));
        A.alpha[i] = (float)alpha;
    }
    double Tm[D * D], Bm[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) Bm[k] = (double)A.B[(int64_t)k * n + i];
    mm<D>(P, Bm, Tm);
    const float4 xv = A.XV[i];
    const double vol = (double)volof32<D>(xv);
    float tt[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) tt[k] = (float)(Tm[k] * vol);
    dstore32<D>(A.T, n, i, tt, xv);
}

// k_solid_accel_csr in fp32; E_k and |a|max partials in fp64
template <int D, int G, bool C16 = false>
__global__ void __launch_bounds__(256) k32_accel_csr(Solid32Args A) {
    using V_t = typename VTR<D, float>::T;
    __shared__ double sh[32];
    const Ctrl *c = A.ctrl;
    if (c->done) return;
    const float dt = (float)c->dt;
    const int64_t n = A.n;
    const int sub = threadIdx.x % G;
    double ek = 0.0, a2m = 0.0;
    for (int it = 0; it < G; ++it) {
        const int64_t i = (int64_t)blockIdx.x * 256 + it * (256 / G) + threadIdx.x / G;
        const bool act = i < n;
        float acc[D];
#pragma unroll
        for (int k = 0; k < D; ++k) acc[k] = 0.f;
        if (act) {
            float xa[3];
            xget32<D>(__ldg(A.XV + i), xa);
            auto visit = [&](int32_t b) {
                float xb[3], Tb[D * D], rel[D], g[D];
                dload32<D>(A.T, n, A.XV, b, Tb, xb);
#pragma unroll
                for (int q = 0; q < D; ++q) rel[q] = xb[q] - xa[q];
                grad_w32<D>(rel, A.ks, g);
#pragma unroll
                for (int r = 0; r < D; ++r)
#pragma unroll
                    for (int cc = 0; cc < D; ++cc) acc[r] = fmaf(Tb[r * D + cc], g[cc], acc[r]);
            };
            if constexpr (C16) {
                walk_chunks<G, true>(A.cptr, A.csr16, i, sub, visit);
            } else {
                const int64_t k1 = A.indptr[i + 1];
                for (int64_t k = A.indptr[i] + sub; k < k1; k += G) visit(__ldg(A.csr + k));
            }
        }
        group_sum32<G>(acc);
        if (act && sub == 0) {
            float Ta[D * D], xd[3];
            dload32<D>(A.T, n, A.XV, i, Ta, xd);
            const float rho0 = A.rho0[i], vola = volof32<D>(__ldg(A.XV + i));
#pragma unroll
            for (int k = 0; k < D; ++k) {
                float ta = 0.f;
#pragma unroll
                for (int cc = 0; cc < D; ++cc) ta += Ta[k * D + cc] * A.G[(int64_t)cc * n + i];
                acc[k] = (acc[k] + ta / vola) / rho0;
                A.a[(int64_t)k * n + i] = acc[k];
            }
            if (A.flags[i] & FL_MOVABLE) {
                V_t *V = reinterpret_cast<V_t *>(A.V);
                float v[3];
                vget(V[i], v);
                double v2 = 0.0, aa = 0.0;
#pragma unroll
                for (int k = 0; k < D; ++k) {
                    v[k] += 0.5f * dt * acc[k];
                    v2 += (double)v[k] * v[k];
                    aa += (double)acc[k] * acc[k];
                }
                V_t w2;
                vset(w2, v);
                V[i] = w2;
                ek += (double)A.mass[i] * v2;
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

// k_solid_vmax in fp32 storage
template <int D>
__global__ void __launch_bounds__(256) k32_vmax(Solid32Args A, int with_accel) {
    using V_t = typename VTR<D, float>::T;
    __shared__ double sh[32];
    if (!with_accel && A.ctrl->done) return;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double v2 = 0.0, a2 = 0.0;
    if (i < A.n) {
        float v[3];
        vget(reinterpret_cast<const V_t *>(A.V)[i], v);
#pragma unroll
        for (int k = 0; k < D; ++k) v2 += (double)v[k] * v[k];
        if (with_accel && (A.flags[i] & FL_MOVABLE)) {
#pragma unroll
            for (int k = 0; k < D; ++k) {
                const double q = A.a[(int64_t)k * A.n + i];
                a2 += q * q;
            }
        }
    }
    const double mv = block_max<256>(v2, sh);
    const double ma = block_max<256>(a2, sh);
    if (threadIdx.x == 0) {
        A.part[2 * A.nblk + blockIdx.x] = mv;
        if (with_accel) A.part[A.nblk + blockIdx.x] = ma;
    }
}

// ---------------------------------------------------- precision switch

// fp64 state -> fp32 state (to32 = 1) or back (to32 = 0).  X (the
// reference position) is the fp64 XV, so u and x convert exactly up to the
// fp32 rounding of u.
template <int D>
__global__ void __launch_bounds__(256) k32_convert(SolidArgs S, Solid32Args A, int to32) {
    using V64 = typename VT<D>::T;
    using V32 = typename VTR<D, float>::T;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n = S.n;
    if (i >= n) return;
    double X[3];
    xget<D>(S.XV[i], X);
    V64 *v64 = reinterpret_cast<V64 *>(S.V);
    V32 *v32 = reinterpret_cast<V32 *>(A.V);
    if (to32) {
        double v[3];
        float w[3];
        vget(v64[i], v);
#pragma unroll
        for (int k = 0; k < D; ++k) w[k] = (float)v[k];
        V32 o;
        vset(o, w);
        v32[i] = o;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            A.u[k * n + i] = (float)(S.x[k * n + i] - X[k]);
            A.a[k * n + i] = (float)S.a[k * n + i];
        }
#pragma unroll
        for (int k = 0; k < D * D; ++k) {
            const double id = (k % (D + 1) == 0) ? 1.0 : 0.0;
            A.H[k * n + i] = (float)(S.F[k * n + i] - id);
            A.Hc[k * n + i] = (float)(S.cp[k * n + i] - id);
        }
        A.alpha[i] = (float)S.alpha[i];
    } else {
        float w[3];
        double v[3] = {0, 0, 0};
        vget(v32[i], w);
#pragma unroll
        for (int k = 0; k < D; ++k) v[k] = w[k];
        V64 o;
        vset(o, v);
        v64[i] = o;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            S.x[k * n + i] = X[k] + (double)A.u[k * n + i];
            S.a[k * n + i] = (double)A.a[k * n + i];
        }
#pragma unroll
        for (int k = 0; k < D * D; ++k) {
            const double id = (k % (D + 1) == 0) ? 1.0 : 0.0;
            S.F[k * n + i] = id + (double)A.H[k * n + i];
            S.cp[k * n + i] = id + (double)A.Hc[k * n + i];
        }
        S.alpha[i] = (double)A.alpha[i];
    }
}

// static fields (reference positions, correction, sum V gradW, masses)
template <int D>
__global__ void __launch_bounds__(256) k32_static(SolidArgs S, Solid32Args A, const double *inv_m, float *inv_m32) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t n = S.n;
    if (i >= n) return;
    const double4 xv = S.XV[i];
    const_cast<float4 *>(A.XV)[i] = make_float4((float)xv.x, (float)xv.y, (float)xv.z, (float)xv.w);
#pragma unroll
    for (int k = 0; k < D * D; ++k) const_cast<float *>(A.B)[k * n + i] = (float)S.B[k * n + i];
#pragma unroll
    for (int k = 0; k < D; ++k) const_cast<float *>(A.G)[k * n + i] = (float)S.G[k * n + i];
    const_cast<float *>(A.mass)[i] = (float)S.mass[i];
    const_cast<float *>(A.rho0)[i] = (float)S.rho0[i];
    inv_m32[i] = (float)inv_m[i];
}

__global__ void k32_narrow(const double *src, float *dst, int64_t m) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < m) dst[i] = (float)src[i];
}

}  // namespace mtsph
