// layer1.cuh -- kernels behind the _accel.py drop-in entry points.
//
// Reference data layout: numpy C order, vectors (n,d), tensors (n,d,d),
// CSR indptr/idx int64 with stored kernel gradients (nnz,d).  One thread
// per particle, neighbours summed in CSR order (the reference's order),
// so results differ from the numba loops only by FMA contraction.
#pragma once

#include "common.cuh"

namespace mtsph {

template <int D>
__global__ void k_l1_velgrad(int64_t n, const double *__restrict__ src, const int64_t *__restrict__ ip,
                             const int64_t *__restrict__ idx, const double *__restrict__ grad,
                             const double *__restrict__ vol, double *out) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    double acc[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) acc[k] = 0.0;
    for (int64_t k = ip[a]; k < ip[a + 1]; ++k) {
        const int64_t b = idx[k];
        const double vb = vol[b];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            const double dv = vb * (src[b * D + r] - src[a * D + r]);
#pragma unroll
            for (int c = 0; c < D; ++c) acc[r * D + c] += dv * grad[k * D + c];
        }
    }
#pragma unroll
    for (int k = 0; k < D * D; ++k) out[a * D * D + k] = acc[k];
}

// out[a] (=|+=) sum_b vol_b (t_a + t_b) . (map_a grad)   (map = I if null)
template <int D>
__global__ void k_l1_pairdiv(int64_t n, const double *__restrict__ tens, const double *__restrict__ amap,
                             const int64_t *__restrict__ ip, const int64_t *__restrict__ idx,
                             const double *__restrict__ grad, const double *__restrict__ vol, double *out,
                             int accumulate) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    double acc[D], ta[D * D], ma[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) {
        ta[k] = tens[a * D * D + k];
        ma[k] = amap ? amap[a * D * D + k] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = accumulate ? out[a * D + k] : 0.0;
    for (int64_t k = ip[a]; k < ip[a + 1]; ++k) {
        const int64_t b = idx[k];
        double g[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            if (amap) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < D; ++c) s += ma[r * D + c] * grad[k * D + c];
                g[r] = s;
            } else {
                g[r] = grad[k * D + r];
            }
        }
        const double vb = vol[b];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) s += (ta[r * D + c] + tens[b * D * D + r * D + c]) * g[c];
            acc[r] += vb * s;
        }
    }
#pragma unroll
    for (int k = 0; k < D; ++k) out[a * D + k] = acc[k];
}

template <int D>
__global__ void k_l1_sdflux(int64_t n, const double *__restrict__ sat, const double *__restrict__ coeff,
                            const double *__restrict__ amap, const int64_t *__restrict__ ip,
                            const int64_t *__restrict__ idx, const double *__restrict__ vol,
                            const double *__restrict__ grad, double *out) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    double acc[D], ma[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) ma[k] = amap[a * D * D + k];
#pragma unroll
    for (int k = 0; k < D; ++k) acc[k] = 0.0;
    for (int64_t k = ip[a]; k < ip[a + 1]; ++k) {
        const int64_t b = idx[k];
        const double w = vol[b] * (sat[a] - sat[b]);
#pragma unroll
        for (int r = 0; r < D; ++r) {
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) s += ma[r * D + c] * grad[k * D + c];
            acc[r] += w * s;
        }
    }
#pragma unroll
    for (int r = 0; r < D; ++r) out[a * D + r] = acc[r] * coeff[a];
}

template <int D>
__global__ void k_l1_pair_w(int64_t np, const double *__restrict__ flux, const double *__restrict__ amap,
                            const int64_t *__restrict__ pi, const int64_t *__restrict__ pj,
                            const double *__restrict__ pg, const double *__restrict__ vol, double *w) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= np) return;
    const int64_t i = pi[k], j = pj[k];
    double acc = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c)
            s += 0.5 * (amap[i * D * D + r * D + c] + amap[j * D * D + r * D + c]) * pg[k * D + c];
        acc += (flux[i * D + r] + flux[j * D + r]) * s;
    }
    w[k] = vol[i] * vol[j] * acc;
}

// out[a] = sum over incident pairs in pair order of (-w if a == i else +w)
__global__ void k_l1_pair_gather(int64_t n, const int64_t *__restrict__ inc_ptr,
                                 const int64_t *__restrict__ inc, const int64_t *__restrict__ pi,
                                 const double *__restrict__ w, double *out) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    double s = 0.0;
    for (int64_t m = inc_ptr[a]; m < inc_ptr[a + 1]; ++m) {
        const int64_t k = inc[m];
        s = (pi[k] == a) ? s - w[k] : s + w[k];
    }
    out[a] = s;
}

template <int D>
__global__ void k_l1_porous_tbuf(int64_t n, const double *__restrict__ F, const double *__restrict__ p,
                                 const double *__restrict__ corr, double mu, double lam, double *tbuf,
                                 double *jout, int *bad) {
    const int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (a >= n) return;
    double f[D * D], t[D * D];
#pragma unroll
    for (int k = 0; k < D * D; ++k) f[k] = F[a * D * D + k];
    const double j = det_d<D>(f);
    jout[a] = j;
    if (!(j > 0.0)) {
#pragma unroll
        for (int k = 0; k < D * D; ++k) tbuf[a * D * D + k] = 0.0;
        atomicAdd(bad, 1);
        return;
    }
    double fi[D * D], e[D * D], sg[D * D], pm[D * D], cb[D * D];
    inv_d<D>(f, j, fi);
    double tre = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
#pragma unroll
        for (int c = 0; c < D; ++c) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k) s += fi[k * D + r] * fi[k * D + c];
            e[r * D + c] = -0.5 * s;
        }
        e[r * D + r] += 0.5;
        tre += e[r * D + r];
    }
    const double dia = lam * tre - p[a];
#pragma unroll
    for (int k = 0; k < D * D; ++k) sg[k] = 2.0 * mu * e[k];
#pragma unroll
    for (int r = 0; r < D; ++r) sg[r * D + r] += dia;
    mmt<D>(sg, fi, pm);
#pragma unroll
    for (int k = 0; k < D * D; ++k) { pm[k] *= j; cb[k] = corr[a * D * D + k]; }
    mm<D>(pm, cb, t);
#pragma unroll
    for (int k = 0; k < D * D; ++k) tbuf[a * D * D + k] = t[k];
}

// reference damping arrays, level-scheduled exact serial sweep
struct L1Sweep {
    double *vel;
    const int64_t *pi, *pj, *gptr, *gscr, *level_ptr, *level_groups;
    const double *pd, *imi, *imj;
    double *scratch;
    int64_t nlevels;
};

template <int D> __device__ void l1_visit(const L1Sweep &S, int64_t g, double half) {
    const int64_t lo = S.gptr[g], hi = S.gptr[g + 1];
    double *vel = S.vel;
    if (hi - lo == 1) {
        const double c = half * S.pd[lo];
        const double ca = c * S.imi[lo], cb = c * S.imj[lo];
        const int64_t a = S.pi[lo], b = S.pj[lo];
        const double den = 1.0 + ca + cb;
#pragma unroll
        for (int m = 0; m < D; ++m) {
            const double u = (vel[a * D + m] - vel[b * D + m]) / den;
            vel[a * D + m] -= ca * u;
            vel[b * D + m] += cb * u;
        }
        return;
    }
    double *Sc = S.scratch + S.gscr[g];
    const int nbmax = (int)(2 * (hi - lo));
    double *Am = Sc, *rhs = Sc + nbmax * nbmax;
    long long *loc = reinterpret_cast<long long *>(rhs + 3 * nbmax);
    int nb = 0;
    for (int64_t k = lo; k < hi; ++k) {
        const int64_t e[2] = {S.pi[k], S.pj[k]};
        for (int s = 0; s < 2; ++s) {
            bool found = false;
            for (int t = 0; t < nb; ++t) if (loc[t] == e[s]) { found = true; break; }
            if (!found) loc[nb++] = e[s];
        }
    }
    for (int r = 0; r < nb; ++r) {
        for (int c = 0; c < nb; ++c) Am[r * nb + c] = (r == c) ? 1.0 : 0.0;
        for (int m = 0; m < D; ++m) rhs[r * 3 + m] = vel[loc[r] * D + m];
    }
    for (int64_t k = lo; k < hi; ++k) {
        const double c = half * S.pd[k];
        int ia = 0, ib = 0;
        for (int t = 0; t < nb; ++t) {
            if (loc[t] == S.pi[k]) ia = t;
            if (loc[t] == S.pj[k]) ib = t;
        }
        const double ca = c * S.imi[k], cb = c * S.imj[k];
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
        for (int m = 0; m < D; ++m) vel[loc[t] * D + m] = rhs[t * 3 + m];
}

template <int D> __global__ void __launch_bounds__(1024) k_l1_sweep(L1Sweep S, double half) {
    for (int64_t L = 0; L < S.nlevels; ++L) {
        for (int64_t k = S.level_ptr[L] + threadIdx.x; k < S.level_ptr[L + 1]; k += blockDim.x)
            l1_visit<D>(S, S.level_groups[k], half);
        __syncthreads();
    }
    for (int64_t L = S.nlevels - 1; L >= 0; --L) {
        for (int64_t k = S.level_ptr[L] + threadIdx.x; k < S.level_ptr[L + 1]; k += blockDim.x)
            l1_visit<D>(S, S.level_groups[k], half);
        __syncthreads();
    }
}

}  // namespace mtsph
