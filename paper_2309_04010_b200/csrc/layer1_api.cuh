// layer1_api.cuh -- host-pointer drop-ins for the reference's _accel.py
// kernels (included at the end of mtsph_b200.cu).  Each call stages the
// inputs to HBM, runs the sm_100a kernel, and copies the outputs back.
#pragma once

namespace {

template <class F> void dispatch_d(int d, F &&f) {
    if (d == 1) f(std::integral_constant<int, 1>{});
    else if (d == 2) f(std::integral_constant<int, 2>{});
    else if (d == 3) f(std::integral_constant<int, 3>{});
    else throw Error(MTSPH_ERR_ARG, "dimension must be 1, 2 or 3");
}

template <class T> DBuf<T> up(const T *h, size_t n) {
    DBuf<T> b(n ? n : 1);
    if (n) MT_CUDA(cudaMemcpy(b.p, h, n * sizeof(T), cudaMemcpyHostToDevice));
    return b;
}
template <class T> void down(T *h, const DBuf<T> &b, size_t n) {
    if (n) MT_CUDA(cudaMemcpy(h, b.p, n * sizeof(T), cudaMemcpyDeviceToHost));
}

int64_t csr_nnz(int64_t n, const int64_t *indptr) { return indptr[n]; }

}  // namespace

extern "C" mtsph_status mtsph_velocity_gradient_gather(int64_t n, int d, const double *src, const int64_t *indptr,
                                                       const int64_t *idx, const double *grad, const double *vol,
                                                       double *out) {
    API_BEGIN
    require_device();
    const int64_t nnz = csr_nnz(n, indptr);
    auto dsrc = up(src, n * d);
    auto dgr = up(grad, nnz * d);
    auto dvol = up(vol, n);
    auto dip = up(indptr, n + 1);
    auto didx = up(idx, nnz);
    DBuf<double> dout(n * d * d);
    dispatch_d(d, [&](auto D) {
        k_l1_velgrad<decltype(D)::value><<<blocks_for(n), 256>>>(n, dsrc.p, dip.p, didx.p, dgr.p, dvol.p, dout.p);
    });
    MT_LAUNCH_CHECK();
    down(out, dout, n * d * d);
    API_END
}

static void pairdiv_common(int64_t n, int d, const double *tens, const double *amap, const int64_t *indptr,
                           const int64_t *idx, const double *grad, const double *vol, double *out, int acc) {
    require_device();
    const int64_t nnz = csr_nnz(n, indptr);
    auto dt = up(tens, n * d * d);
    auto dgr = up(grad, nnz * d);
    auto dvol = up(vol, n);
    auto dip = up(indptr, n + 1);
    auto didx = up(idx, nnz);
    DBuf<double> dmap;
    if (amap) dmap = up(amap, n * d * d);
    auto dout = acc ? up(out, n * d) : DBuf<double>(n * d);
    dispatch_d(d, [&](auto D) {
        k_l1_pairdiv<decltype(D)::value><<<blocks_for(n), 256>>>(n, dt.p, amap ? dmap.p : nullptr, dip.p, didx.p,
                                                                 dgr.p, dvol.p, dout.p, acc);
    });
    MT_LAUNCH_CHECK();
    down(out, dout, n * d);
}

extern "C" mtsph_status mtsph_pair_tensor_divergence(int64_t n, int d, const double *tens, const int64_t *indptr,
                                                     const int64_t *idx, const double *grad, const double *vol,
                                                     double *out) {
    API_BEGIN
    pairdiv_common(n, d, tens, nullptr, indptr, idx, grad, vol, out, 0);
    API_END
}

extern "C" mtsph_status mtsph_pair_tensor_divergence_mapped(int64_t n, int d, const double *tens, const double *amap,
                                                            const int64_t *indptr, const int64_t *idx,
                                                            const double *grad, const double *vol, double *out) {
    API_BEGIN
    if (!amap) throw Error(MTSPH_ERR_ARG, "amap required");
    pairdiv_common(n, d, tens, amap, indptr, idx, grad, vol, out, 1);
    API_END
}

extern "C" mtsph_status mtsph_scalar_difference_flux(int64_t n, int d, const double *sat, const double *coeff,
                                                     const double *amap, const int64_t *indptr, const int64_t *idx,
                                                     const double *vol, const double *grad, double *out) {
    API_BEGIN
    require_device();
    const int64_t nnz = csr_nnz(n, indptr);
    auto ds = up(sat, n);
    auto dc = up(coeff, n);
    auto dm = up(amap, n * d * d);
    auto dvol = up(vol, n);
    auto dgr = up(grad, nnz * d);
    auto dip = up(indptr, n + 1);
    auto didx = up(idx, nnz);
    DBuf<double> dout(n * d);
    dispatch_d(d, [&](auto D) {
        k_l1_sdflux<decltype(D)::value><<<blocks_for(n), 256>>>(n, ds.p, dc.p, dm.p, dip.p, didx.p, dvol.p, dgr.p,
                                                                dout.p);
    });
    MT_LAUNCH_CHECK();
    down(out, dout, n * d);
    API_END
}

extern "C" mtsph_status mtsph_conservative_mass_rate(int64_t n, int d, const double *flux, const double *amap,
                                                     int64_t npairs, const int64_t *pair_i, const int64_t *pair_j,
                                                     const double *pair_grad, const double *vol, double *out) {
    API_BEGIN
    require_device();
    // incidence lists in pair order (host, O(npairs)) -> deterministic
    // gather with the reference's accumulation order
    std::vector<int64_t> ptr(n + 1, 0), inc(2 * npairs);
    for (int64_t k = 0; k < npairs; ++k) { ptr[pair_i[k] + 1]++; ptr[pair_j[k] + 1]++; }
    for (int64_t a = 0; a < n; ++a) ptr[a + 1] += ptr[a];
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    for (int64_t k = 0; k < npairs; ++k) { inc[fill[pair_i[k]]++] = k; inc[fill[pair_j[k]]++] = k; }
    auto df = up(flux, n * d);
    auto dm = up(amap, n * d * d);
    auto dpi = up(pair_i, npairs);
    auto dpj = up(pair_j, npairs);
    auto dpg = up(pair_grad, npairs * d);
    auto dvol = up(vol, n);
    auto dptr = up(ptr.data(), n + 1);
    auto dinc = up(inc.data(), 2 * npairs);
    DBuf<double> w(npairs ? npairs : 1), dout(n);
    dispatch_d(d, [&](auto D) {
        if (npairs)
            k_l1_pair_w<decltype(D)::value><<<blocks_for(npairs), 256>>>(npairs, df.p, dm.p, dpi.p, dpj.p, dpg.p,
                                                                         dvol.p, w.p);
    });
    k_l1_pair_gather<<<blocks_for(n), 256>>>(n, dptr.p, dinc.p, dpi.p, w.p, dout.p);
    MT_LAUNCH_CHECK();
    down(out, dout, n);
    API_END
}

extern "C" mtsph_status mtsph_porous_stress_rhs(int64_t n, int d, const double *def_grad, const double *pressure,
                                                const double *corr, const int64_t *indptr, const int64_t *idx,
                                                const double *grad0, const double *vol0, double mu, double lam,
                                                double *tbuf, double *out_j, double *out_rate) {
    API_BEGIN
    require_device();
    const int64_t nnz = csr_nnz(n, indptr);
    auto dF = up(def_grad, n * d * d);
    auto dp = up(pressure, n);
    auto dc = up(corr, n * d * d);
    auto dip = up(indptr, n + 1);
    auto didx = up(idx, nnz);
    auto dgr = up(grad0, nnz * d);
    auto dvol = up(vol0, n);
    DBuf<double> dt(n * d * d), dj(n), dr(n * d);
    DBuf<int> bad(1);
    bad.zero();
    dispatch_d(d, [&](auto D) {
        constexpr int DD = decltype(D)::value;
        k_l1_porous_tbuf<DD><<<blocks_for(n), 256>>>(n, dF.p, dp.p, dc.p, mu, lam, dt.p, dj.p, bad.p);
        k_l1_pairdiv<DD><<<blocks_for(n), 256>>>(n, dt.p, nullptr, dip.p, didx.p, dgr.p, dvol.p, dr.p, 0);
    });
    MT_LAUNCH_CHECK();
    down(tbuf, dt, n * d * d);
    down(out_j, dj, n);
    down(out_rate, dr, n * d);
    API_END
}

extern "C" mtsph_status mtsph_damping_sweep(int64_t n, int d, double *vel, int64_t npairs, const int64_t *pair_i,
                                            const int64_t *pair_j, const double *pair_damp, const double *inv_mass_i,
                                            const double *inv_mass_j, int64_t ngroups, const int64_t *group_ptr,
                                            double eta, double dt) {
    API_BEGIN
    require_device();
    if (eta < 0.0) throw Error(MTSPH_ERR_ARG, "eta must be >= 0");
    if (npairs == 0 || ngroups == 0) return MTSPH_OK;
    // level schedule of the serial group order + scratch for group solves
    std::vector<int32_t> last(n, 0), lev(ngroups);
    std::vector<int64_t> scr(ngroups + 1, 0);
    int32_t maxl = 0;
    for (int64_t g = 0; g < ngroups; ++g) {
        const int64_t lo = group_ptr[g], hi = group_ptr[g + 1];
        if (hi - lo > 64) throw Error(MTSPH_ERR_GEOMETRY, "more than 64 pairs in one damping group");
        int32_t L = 0;
        for (int64_t k = lo; k < hi; ++k) L = std::max(L, std::max(last[pair_i[k]], last[pair_j[k]]));
        ++L;
        for (int64_t k = lo; k < hi; ++k) last[pair_i[k]] = last[pair_j[k]] = L;
        lev[g] = L;
        maxl = std::max(maxl, L);
        const int64_t nb = 2 * (hi - lo);
        scr[g + 1] = scr[g] + (hi - lo > 1 ? nb * nb + 4 * nb : 0);
    }
    std::vector<int64_t> lptr(maxl + 1, 0), lg(ngroups);
    for (int64_t g = 0; g < ngroups; ++g) lptr[lev[g]]++;
    for (int32_t L = 1; L <= maxl; ++L) lptr[L] += lptr[L - 1];
    std::vector<int64_t> fillp(lptr.begin(), lptr.end() - 1);
    for (int64_t g = 0; g < ngroups; ++g) lg[fillp[lev[g] - 1]++] = g;
    auto dv = up(vel, n * d);
    auto dpi = up(pair_i, npairs);
    auto dpj = up(pair_j, npairs);
    auto dgp = up(group_ptr, ngroups + 1);
    auto dpd = up(pair_damp, npairs);
    auto dmi = up(inv_mass_i, npairs);
    auto dmj = up(inv_mass_j, npairs);
    auto dscr_off = up(scr.data(), ngroups + 1);
    auto dlp = up(lptr.data(), maxl + 1);
    auto dlg = up(lg.data(), ngroups);
    DBuf<double> scratch(std::max<int64_t>(scr[ngroups], 1));
    L1Sweep S{dv.p, dpi.p, dpj.p, dgp.p, dscr_off.p, dlp.p, dlg.p, dpd.p, dmi.p, dmj.p, scratch.p, maxl};
    const double half = 0.5 * dt * eta;
    dispatch_d(d, [&](auto D) { k_l1_sweep<decltype(D)::value><<<1, 1024>>>(S, half); });
    MT_LAUNCH_CHECK();
    down(vel, dv, n * d);
    API_END
}
