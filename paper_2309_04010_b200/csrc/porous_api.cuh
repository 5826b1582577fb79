// porous_api.cuh -- C ABI of the device-resident porous membrane
// (included at the end of mtsph_b200.cu; shares its error plumbing).
#pragma once

struct mtsph_porous {
    NbhDev nb;
    int d = 0;
    int64_t n = 0;
    cudaStream_t s = nullptr;
    DBuf<unsigned char> V;
    DBuf<double> x, F, M, q, vl, rate, frate, mass_l, sat, pres, J, rho_lf, mix, inv_mix, volc, coeff,
        amap, mrate, T, G, part, rm, rf;
    DBuf<uint8_t> flags;
    DBuf<Ctrl> ctrl;
    DBuf<int64_t> level_ptr;
    TiledSched tiled;
    Ctrl *hc = nullptr;
    PorMat m{};
    double contact_time = 0.0, evap = 0.0;
    int nblk = 0;
    double outer_dt = 0.0, outer_t = 0.0;   // multi-rank outer phases
    std::vector<int64_t> iperm_h;           // original -> internal (pack/unpack)
    int64_t launches = 0;
    int per_step_launches = 0;
    cudaGraphExec_t graphs[3] = {nullptr, nullptr, nullptr};
    int graph_steps[3] = {4, 32, 128};
    cudaEvent_t ev_outer[2] = {nullptr, nullptr};   // brackets the last advance_slow
    ~mtsph_porous() {
        for (auto e : ev_outer) if (e) cudaEventDestroy(e);
        for (auto &g : graphs) if (g) cudaGraphExecDestroy(g);
        if (hc) cudaFreeHost(hc);
        if (s) cudaStreamDestroy(s);
    }
    PorousArgs args() {
        PorousArgs A{};
        A.n = n; A.XV = nb.XV.p; A.V = V.p;
        A.x = x.p; A.F = F.p; A.M = M.p; A.q = q.p; A.vl = vl.p; A.rate = rate.p; A.frate = frate.p;
        A.mass_l = mass_l.p; A.sat = sat.p; A.pres = pres.p; A.J = J.p; A.rho_lf = rho_lf.p;
        A.mix = mix.p; A.inv_mix = inv_mix.p; A.volc = volc.p; A.coeff = coeff.p; A.amap = amap.p;
        A.mrate = mrate.p; A.T = T.p; A.G = G.p; A.rm = rm.p; A.rf = rf.p; A.B = nb.B.p; A.flags = flags.p; A.indptr = nb.indptr.p;
        A.csr = nb.csr.p; A.cptr = nb.cptr.p; A.csr16 = nb.csr16.p; A.mag16 = nb.mag16.p; A.perm = nb.perm.p; A.part = part.p; A.nblk = nblk;
        A.ctrl = ctrl.p; A.ks = nb.ks; A.m = m;
        return A;
    }
    SweepArgs sweep_args() {
        SweepArgs S{};
        S.pi = nb.pi.p; S.pj = nb.pj.p; S.gptr = nb.gptr.p; S.gscr = nb.gscr.p;
        S.scratch = nb.scratch.p; S.XV = nb.XV.p; S.inv_m = inv_mix.p; S.V = V.p; S.ks = nb.ks;
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

template <int D> static int porous_step(mtsph_porous *P, int mode) {
    PorousArgs A = P->args();
    const unsigned nb = blocks_for(P->n);
    k_por_kick1<D><<<nb, 256, 0, P->s>>>(A);
    k_por_stress<D><<<nb, 256, 0, P->s>>>(A);
    k_por_constit<D><<<nb, 256, 0, P->s>>>(A);
    k_por_accel<D><<<nb, 256, 0, P->s>>>(A);
    MT_LAUNCH_CHECK();
    int l = 4;
    if (P->nb.sweep == 3) {
        TiledArgs T{P->tiled.range_off.p, P->tiled.ranges.p, P->tiled.halo_n.p, P->tiled.pair_off.p,
                    P->tiled.pairs.p, P->tiled.pd.p, P->tiled.sub_off.p, P->tiled.sub.p, P->inv_mix.p, P->V.p,
                    P->tiled.maxsub, P->tiled.hid_off.p, P->tiled.hid.p};
        l += launch_tiled_sweep<D>(P->tiled, T, P->ctrl.p, P->s);
    } else {
        l += launch_sweep<D>(P->nb, P->sweep_args(), P->level_ptr.p, P->ctrl.p, P->s);
    }
    k_por_post_step<D><<<nb, 256, 0, P->s>>>(A, 0);
    k_ctrl<<<1, kCtrlThreads, 0, P->s>>>(P->ctrl.p, P->part.p, P->nblk, mode);
    MT_LAUNCH_CHECK();
    return l + 2;
}

static int porous_step_any(mtsph_porous *P, int mode) {
    return P->d == 2 ? porous_step<2>(P, mode) : porous_step<3>(P, mode);
}

template <int D> static void porous_init_dt(mtsph_porous *P) {
    PorousArgs A = P->args();
    k_por_post_step<D><<<blocks_for(P->n), 256, 0, P->s>>>(A, 1);
    k_ctrl<<<1, kCtrlThreads, 0, P->s>>>(P->ctrl.p, P->part.p, P->nblk, CTRL_INIT);
    MT_LAUNCH_CHECK();
    P->launches += 2;
}

static void check_porous_errors(mtsph_porous *P) {
    if (P->hc->err_inv != ~0ull)
        throw Error(MTSPH_ERR_INVERSION, "non-positive deformation determinant (first id " +
                                             std::to_string(P->hc->err_inv) + ")",
                    {(int64_t)P->hc->err_inv});
    if (P->hc->remote_err)
        throw Error(MTSPH_ERR_NONFINITE, "inner loop stopped by an error on another rank");
}

extern "C" mtsph_status mtsph_porous_create(const mtsph_porous_desc *dsc, mtsph_porous **out) {
    API_BEGIN
    require_device();
    const int64_t n = dsc->n;
    const int d = dsc->d;
    if (d != 2 && d != 3) throw Error(MTSPH_ERR_ARG, "porous problems support d = 2 or 3");
    auto P = std::make_unique<mtsph_porous>();
    P->n = n;
    P->d = d;
    MT_CUDA(cudaStreamCreateWithFlags(&P->s, cudaStreamNonBlocking));
    if (dsc->grid) {
        P->nb.has_grid = true;
        for (int k = 0; k < 3; ++k) {
            P->nb.grid_lo[k] = dsc->grid[k];
            P->nb.grid_hi[k] = dsc->grid[3 + k];
        }
    }
    if (dsc->ghost && dsc->sweep != 3) throw Error(MTSPH_ERR_ARG, "ghost particles (multi-rank) need the tiled sweep");
    if (dsc->ghost) {
        // as mtsph_solid_create: ghost flags in the internal order feed the
        // tiled schedule, so the schedule waits for the neighbour build
        P->nb.ghost_orig = dsc->ghost;
        build_nbh(P->nb, n, d, dsc->pos, dsc->vol, dsc->h_axes, 0, P->s);
        P->nb.ghost_orig = nullptr;
        P->nb.sweep = dsc->sweep;
        std::vector<int64_t> pm(n);
        P->nb.perm.download(pm.data(), n, P->s);
        MT_CUDA(cudaStreamSynchronize(P->s));
        P->nb.ghost_internal.resize(n);
        for (int64_t k = 0; k < n; ++k) P->nb.ghost_internal[k] = dsc->ghost[pm[k]] ? 1 : 0;
    } else {
        build_nbh(P->nb, n, d, dsc->pos, dsc->vol, dsc->h_axes, dsc->sweep, P->s);
    }
    build_chunked(P->nb, kPorLanes, P->s, true, true);
    if (dsc->sweep == 3) build_tiled_auto(P->nb, P->tiled, P->s, dsc->tile);
    std::vector<int64_t> perm(n);
    P->nb.perm.download(perm.data(), n, P->s);
    MT_CUDA(cudaStreamSynchronize(P->s));
    const int dd = d * d;
    std::vector<double> x((size_t)d * n), F((size_t)dd * n, 0.0), mix(n), inv(n), ones(n, 1.0);
    std::vector<uint8_t> flags(n);
    double vol_movable = 0.0;
    for (int64_t k = 0; k < n; ++k) {
        const int64_t o = perm[k];
        for (int c = 0; c < d; ++c) x[(size_t)c * n + k] = dsc->pos[o * d + c];
        for (int c = 0; c < d; ++c) F[(size_t)(c * d + c) * n + k] = 1.0;
        const bool movable = !dsc->constrained[o];
        flags[k] = (movable ? PF_MOVABLE : 0) | ((dsc->contact && dsc->contact[o]) ? PF_CONTACT : 0) |
                   ((dsc->ghost && dsc->ghost[o]) ? PF_GHOST : 0);
        mix[k] = dsc->density0 * dsc->vol[o];
        inv[k] = movable ? 1.0 / mix[k] : 0.0;
    }
    // the reference sums the free volumes in original order
    for (int64_t o = 0; o < n; ++o) if (!dsc->constrained[o]) vol_movable += dsc->vol[o];
    const size_t vbytes = (size_t)n * (d == 3 ? sizeof(double4) : sizeof(double2));
    P->V.alloc(vbytes);
    P->V.zero(P->s);
    P->x.upload(x.data(), x.size(), P->s);
    P->F.upload(F.data(), F.size(), P->s);
    for (DBuf<double> *b : {&P->M, &P->q, &P->vl, &P->rate, &P->frate}) {
        b->alloc((size_t)d * n);
        b->zero(P->s);
    }
    for (DBuf<double> *b : {&P->mass_l, &P->sat, &P->pres, &P->rho_lf, &P->volc, &P->coeff, &P->mrate}) {
        b->alloc(n);
        b->zero(P->s);
    }
    P->J.upload(ones.data(), n, P->s);
    P->mix.upload(mix.data(), n, P->s);
    P->inv_mix.upload(inv.data(), n, P->s);
    P->amap.alloc((size_t)dd * n);
    P->amap.zero(P->s);
    P->rm.alloc((size_t)4 * (d == 3 ? PorRM<3>::planes : PorRM<2>::planes) * n);
    P->rf.alloc((size_t)8 * n);
    P->T.alloc((size_t)n * (d == 3 ? DS<3>::n : DS<2>::n));
    P->T.zero(P->s);
    P->flags.upload(flags.data(), n, P->s);
    P->nblk = (int)blocks_for(n);
    P->part.alloc((size_t)3 * P->nblk);
    P->G.alloc((size_t)d * n);  // static sum_b V_b gradW_ab
    if (d == 2) k_por_gsum<2><<<blocks_for(n), 256, 0, P->s>>>(P->args(), P->G.p);
    else k_por_gsum<3><<<blocks_for(n), 256, 0, P->s>>>(P->args(), P->G.p);
    MT_LAUNCH_CHECK();
    P->part.zero(P->s);
    if (P->nb.sweep == 1) {
        P->level_ptr.upload(P->nb.level_ptr_h.data(), P->nb.level_ptr_h.size(), P->s);
        if (d == 2) build_serial_entries<2>(P->nb, P->sweep_args(), P->s);
        else build_serial_entries<3>(P->nb, P->sweep_args(), P->s);
    }
    PorMat &m = P->m;
    m.rho_s0 = dsc->density0;
    m.D = dsc->diffusivity;
    m.C = dsc->pressure_coeff;
    m.mu = dsc->shear_modulus;
    m.lam = dsc->lame_lambda;
    m.porosity = dsc->porosity;
    m.rho_l0 = dsc->fluid_density0;
    m.sat0 = dsc->initial_saturation;
    P->contact_time = dsc->contact_time;
    P->evap = dsc->evaporation_rate;
    MT_CUDA(cudaMallocHost(&P->hc, sizeof(Ctrl)));
    std::memset(P->hc, 0, sizeof(Ctrl));
    P->hc->h = P->nb.ks.h_min;
    P->hc->sound = std::sqrt(dsc->bulk_modulus / dsc->density0);
    P->hc->cfl = 0.6;
    P->hc->min_dt = INFINITY;
    P->hc->err_inv = P->hc->err_rm = ~0ull;
    P->hc->remote_err = 0;
    P->hc->vol_movable = vol_movable;
    P->ctrl.alloc(1);
    P->push_ctrl();
    *out = P.release();
    API_END
}

extern "C" mtsph_status mtsph_porous_destroy(mtsph_porous *p) {
    delete p;
    return MTSPH_OK;
}

template <int D> static int64_t porous_advance(mtsph_porous *P, double dt, double t) {
    PorousArgs A = P->args();
    const unsigned nb = blocks_for(P->n);
    cudaStream_t s = P->s;
    if (!P->ev_outer[0])
        for (auto &e : P->ev_outer) MT_CUDA(cudaEventCreate(&e));
    MT_CUDA(cudaEventRecord(P->ev_outer[0], s));
    k_por_prep<D><<<nb, 256, 0, s>>>(A, 1);
    k_por_flux<D><<<nb, 256, 0, s>>>(A, 1);
    const int contact_on = t <= P->contact_time * (1.0 + 1e-12) ? 1 : 0;
    const double evap_factor = (!contact_on && P->evap > 0.0) ? std::exp(-P->evap * dt) : 1.0;
    k_por_mass<D><<<nb, 256, 0, s>>>(A, dt, contact_on, evap_factor);
    k_por_prep<D><<<nb, 256, 0, s>>>(A, 0);
    k_por_flux<D><<<nb, 256, 0, s>>>(A, 0);
    k_por_post<D><<<nb, 256, 0, s>>>(A);
    k_por_fluxrate<D><<<nb, 256, 0, s>>>(A);
    MT_LAUNCH_CHECK();
    MT_CUDA(cudaEventRecord(P->ev_outer[1], s));
    P->launches += 7;
    std::vector<double> part(P->nblk);
    P->part.download(part.data(), P->nblk, s);
    P->pull_ctrl();
    double c = 0.0;
    for (double v : part) c += v;
    return (int64_t)std::llround(c);
}

extern "C" mtsph_status mtsph_porous_advance_slow(mtsph_porous *P, double dt_outer, double t,
                                                  int64_t *clamped) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_advance_slow: null handle");
    API_BEGIN
    P->pull_ctrl();
    P->hc->err_inv = ~0ull;
    P->hc->remote_err = 0;
    P->push_ctrl();
    *clamped = P->d == 2 ? porous_advance<2>(P, dt_outer, t) : porous_advance<3>(P, dt_outer, t);
    check_porous_errors(P);
    API_END
}

// ---- multi-rank phases
// sync = false: only enqueue (device-controlled loop; reductions stay in
// the per-block partials for mtsph_porous_rank_partials)
template <int D> static void porous_phase(mtsph_porous *P, int phase, int arg, double out[2], bool sync = true) {
    PorousArgs A = P->args();
    const unsigned nb = blocks_for(P->n);
    cudaStream_t s = P->s;
    out[0] = out[1] = 0.0;
    auto partials = [&](int segs) {
        std::vector<double> h((size_t)segs * P->nblk);
        P->part.download(h.data(), h.size(), s);
        MT_CUDA(cudaStreamSynchronize(s));
        return h;
    };
    switch (phase) {
    case MTSPH_POR_KICK: k_por_kick1<D><<<nb, 256, 0, s>>>(A); break;
    case MTSPH_POR_STRESS:
        k_por_stress<D><<<nb, 256, 0, s>>>(A);
        k_por_constit<D><<<nb, 256, 0, s>>>(A);
        break;
    case MTSPH_POR_ACCEL: {
        if (sync) P->part.zero(s);
        k_por_accel<D><<<nb, 256, 0, s>>>(A);
        MT_LAUNCH_CHECK();
        if (!sync) break;
        const auto h = partials(2);
        for (int b = 0; b < P->nblk; ++b) {
            out[0] += h[b];
            out[1] = std::max(out[1], h[P->nblk + b]);
        }
        break;
    }
    case MTSPH_POR_SWEEP: {
        if (P->nb.sweep != 3) throw Error(MTSPH_ERR_ARG, "sweep phases need the tiled schedule");
        const int c = arg & 63, dir = arg >= 64 ? -1 : 1;
        const TiledSched &t = P->tiled;
        if (c + 1 >= (int)t.colour_ptr.size()) throw Error(MTSPH_ERR_ARG, "colour out of range");
        const int64_t t0 = t.colour_ptr[c], t1 = t.colour_ptr[c + 1];
        if (t1 > t0) {
            TiledArgs T{t.range_off.p, t.ranges.p, t.halo_n.p, t.pair_off.p, t.pairs.p, t.pd.p, t.sub_off.p,
                        t.sub.p, P->inv_mix.p, P->V.p, t.maxsub, t.hid_off.p, t.hid.p};
            k_sweep_tiled<D><<<(unsigned)(t1 - t0), t.threads, tiled_smem_bytes(t, D), s>>>(T, t0, dir, P->ctrl.p);
        }
        break;
    }
    case MTSPH_POR_POSTSTEP:
    case MTSPH_POR_AMAX: {
        if (sync) P->part.zero(s);
        k_por_post_step<D><<<nb, 256, 0, s>>>(A, phase == MTSPH_POR_AMAX ? 1 : 0);
        MT_LAUNCH_CHECK();
        if (!sync) break;
        const auto h = partials(3);
        for (int b = 0; b < P->nblk; ++b) {
            out[0] = std::max(out[0], h[2 * P->nblk + b]);
            out[1] = std::max(out[1], h[P->nblk + b]);
        }
        break;
    }
    case MTSPH_POR_PREP_MAP: k_por_prep<D><<<nb, 256, 0, s>>>(A, 1); break;
    case MTSPH_POR_FLUX_MASS: k_por_flux<D><<<nb, 256, 0, s>>>(A, 1); break;
    case MTSPH_POR_MASS: {
        const double dt = P->outer_dt, t = P->outer_t;
        const int contact_on = t <= P->contact_time * (1.0 + 1e-12) ? 1 : 0;
        const double evap_factor = (!contact_on && P->evap > 0.0) ? std::exp(-P->evap * dt) : 1.0;
        P->part.zero(s);
        k_por_mass<D><<<nb, 256, 0, s>>>(A, dt, contact_on, evap_factor);
        MT_LAUNCH_CHECK();
        const auto h = partials(1);   // one host read per outer step
        for (int b = 0; b < P->nblk; ++b) out[0] += h[b];
        break;
    }
    case MTSPH_POR_PREP: k_por_prep<D><<<nb, 256, 0, s>>>(A, 0); break;
    case MTSPH_POR_FLUX: k_por_flux<D><<<nb, 256, 0, s>>>(A, 0); break;
    case MTSPH_POR_POST: k_por_post<D><<<nb, 256, 0, s>>>(A); break;
    case MTSPH_POR_FLUXRATE: k_por_fluxrate<D><<<nb, 256, 0, s>>>(A); break;
    default: throw Error(MTSPH_ERR_ARG, "unknown porous phase");
    }
    MT_LAUNCH_CHECK();
    P->launches += 1;
    if (sync) MT_CUDA(cudaStreamSynchronize(s));
}

extern "C" mtsph_status mtsph_porous_set_step(mtsph_porous *P, double dt, double eta) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_set_step: null handle");
    API_BEGIN
    P->pull_ctrl();
    P->hc->dt = dt;
    P->hc->eta = eta;
    P->hc->done = 0;
    P->hc->err_inv = ~0ull;
    P->hc->remote_err = 0;
    P->push_ctrl();
    API_END
}

extern "C" mtsph_status mtsph_porous_set_outer(mtsph_porous *P, double dt_outer, double t) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_set_outer: null handle");
    P->outer_dt = dt_outer;
    P->outer_t = t;
    return MTSPH_OK;
}

extern "C" mtsph_status mtsph_porous_phase(mtsph_porous *P, int phase, int arg, double out[2]) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_phase: null handle");
    API_BEGIN
    if (P->d == 2) porous_phase<2>(P, phase, arg, out); else porous_phase<3>(P, phase, arg, out);
    if (phase == MTSPH_POR_STRESS || phase == MTSPH_POR_PREP_MAP || phase == MTSPH_POR_PREP) {
        P->pull_ctrl();
        check_porous_errors(P);
    }
    API_END
}

static void porous_pack_common(mtsph_porous *P, const char *field, int64_t m, const int64_t *ids, double *host,
                               const double *in, bool pack) {
    const std::string f(field);
    const int which = f == "vel" ? 0 : f == "T" ? 1 : f == "satvol" ? 2 : f == "rm" ? 3 : f == "rf" ? 4
                    : f == "inv_mix" ? 5 : -1;
    if (which < 0) throw Error(MTSPH_ERR_ARG, "porous pack fields: vel, T, satvol, rm, rf, inv_mix");
    if (m <= 0) return;
    if (P->iperm_h.empty()) {
        P->iperm_h.resize(P->n);
        P->nb.iperm.download(P->iperm_h.data(), P->n, P->s);
        MT_CUDA(cudaStreamSynchronize(P->s));
    }
    std::vector<int64_t> internal(m);
    for (int64_t k = 0; k < m; ++k) {
        if (ids[k] < 0 || ids[k] >= P->n) throw Error(MTSPH_ERR_ARG, "particle id out of range");
        internal[k] = P->iperm_h[ids[k]];
    }
    const int w = por_field_width(which, P->d);
    DBuf<int64_t> dids(m);
    DBuf<double> buf((size_t)m * w);
    dids.upload(internal.data(), m, P->s);
    if (!pack) buf.upload(in, (size_t)m * w, P->s);
    PorousArgs A = P->args();
    if (P->d == 2) k_por_pack<2><<<blocks_for(m), 256, 0, P->s>>>(A, m, dids.p, which, w, buf.p, pack ? 0 : 1);
    else k_por_pack<3><<<blocks_for(m), 256, 0, P->s>>>(A, m, dids.p, which, w, buf.p, pack ? 0 : 1);
    MT_LAUNCH_CHECK();
    P->launches += 1;
    if (pack) buf.download(host, (size_t)m * w, P->s);
    MT_CUDA(cudaStreamSynchronize(P->s));
}

extern "C" mtsph_status mtsph_porous_pack(mtsph_porous *P, const char *field, int64_t m, const int64_t *ids,
                                          double *host) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_pack: null handle");
    API_BEGIN
    porous_pack_common(P, field, m, ids, host, nullptr, true);
    API_END
}

extern "C" mtsph_status mtsph_porous_unpack(mtsph_porous *P, const char *field, int64_t m, const int64_t *ids,
                                            const double *host) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_unpack: null handle");
    API_BEGIN
    porous_pack_common(P, field, m, ids, nullptr, host, false);
    API_END
}

extern "C" mtsph_status mtsph_porous_phase_async(mtsph_porous *P, int phase, int arg) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_phase_async: null handle");
    API_BEGIN
    double out[2];
    if (P->d == 2) porous_phase<2>(P, phase, arg, out, false); else porous_phase<3>(P, phase, arg, out, false);
    API_END
}

extern "C" mtsph_status mtsph_porous_begin_loop(mtsph_porous *P, const mtsph_inner_params *p,
                                                double vol_movable) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_begin_loop: null handle");
    API_BEGIN
    P->pull_ctrl();
    Ctrl *c = P->hc;
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
    if (vol_movable > 0.0) c->vol_movable = vol_movable;   // the whole problem's, for E_k
    P->push_ctrl();
    API_END
}

extern "C" mtsph_status mtsph_porous_rank_partials(mtsph_porous *P, int mode, double *dev_out) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_rank_partials: null handle");
    API_BEGIN
    if (mode != CTRL_INIT && mode != CTRL_STEP) throw Error(MTSPH_ERR_ARG, "mode: 0 (initial step) or 1 (step)");
    k_rank_partials<<<1, 256, 0, P->s>>>(P->ctrl.p, P->part.p, P->nblk, mode, dev_out);
    MT_LAUNCH_CHECK();
    P->launches += 1;
    API_END
}

extern "C" mtsph_status mtsph_porous_control_ranks(mtsph_porous *P, const double *dev_gathered, int nranks,
                                                   int mode) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_control_ranks: null handle");
    API_BEGIN
    if (mode != CTRL_INIT && mode != CTRL_STEP) throw Error(MTSPH_ERR_ARG, "mode: 0 (initial step) or 1 (step)");
    if (nranks < 1) throw Error(MTSPH_ERR_ARG, "nranks must be positive");
    k_ctrl_ranks<<<1, 32, 0, P->s>>>(P->ctrl.p, dev_gathered, nranks, mode);
    MT_LAUNCH_CHECK();
    P->launches += 1;
    API_END
}

extern "C" mtsph_status mtsph_porous_loop_state(mtsph_porous *P, mtsph_inner_result *r, int *done) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_loop_state: null handle");
    API_BEGIN
    P->pull_ctrl();
    const Ctrl *c = P->hc;
    *done = c->done;
    r->n_inner = c->n_inner;
    r->cap_hit = c->cap_hit;
    r->ek = c->ek;
    r->min_dt = c->min_dt;
    r->last_dt = c->last_dt;
    check_porous_errors(P);
    API_END
}

extern "C" mtsph_status mtsph_porous_internal_ids(mtsph_porous *P, int64_t m, const int64_t *ids,
                                                  int64_t *internal) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_internal_ids: null handle");
    API_BEGIN
    if (P->iperm_h.empty()) {
        P->iperm_h.resize(P->n);
        P->nb.iperm.download(P->iperm_h.data(), P->n, P->s);
        MT_CUDA(cudaStreamSynchronize(P->s));
    }
    for (int64_t k = 0; k < m; ++k) {
        if (ids[k] < 0 || ids[k] >= P->n) throw Error(MTSPH_ERR_ARG, "particle id out of range");
        internal[k] = P->iperm_h[ids[k]];
    }
    API_END
}

extern "C" mtsph_status mtsph_porous_stream(const mtsph_porous *P, void **stream) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_stream: null handle");
    *stream = (void *)P->s;
    return MTSPH_OK;
}

static int porous_field(const char *field) {
    const std::string f(field ? field : "");
    const int which = f == "vel" ? 0 : f == "T" ? 1 : f == "satvol" ? 2 : f == "rm" ? 3 : f == "rf" ? 4
                    : f == "inv_mix" ? 5 : -1;
    if (which < 0) throw Error(MTSPH_ERR_ARG, "porous pack fields: vel, T, satvol, rm, rf, inv_mix");
    return which;
}

// device-resident exchange: internal ids and the buffer are device memory,
// the kernel is enqueued on the problem's stream (no host synchronisation)
extern "C" mtsph_status mtsph_porous_pack_device(mtsph_porous *P, const char *field, int64_t m,
                                                 const int64_t *ids, double *out) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_pack_device: null handle");
    API_BEGIN
    const int which = porous_field(field);
    if (m <= 0) return MTSPH_OK;
    const int w = por_field_width(which, P->d);
    if (P->d == 2) k_por_pack<2><<<blocks_for(m), 256, 0, P->s>>>(P->args(), m, ids, which, w, out, 0);
    else k_por_pack<3><<<blocks_for(m), 256, 0, P->s>>>(P->args(), m, ids, which, w, out, 0);
    MT_LAUNCH_CHECK();
    P->launches += 1;
    API_END
}

extern "C" mtsph_status mtsph_porous_unpack_device(mtsph_porous *P, const char *field, int64_t m,
                                                   const int64_t *ids, const double *in) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_unpack_device: null handle");
    API_BEGIN
    const int which = porous_field(field);
    if (m <= 0) return MTSPH_OK;
    const int w = por_field_width(which, P->d);
    if (P->d == 2)
        k_por_pack<2><<<blocks_for(m), 256, 0, P->s>>>(P->args(), m, ids, which, w, const_cast<double *>(in), 1);
    else
        k_por_pack<3><<<blocks_for(m), 256, 0, P->s>>>(P->args(), m, ids, which, w, const_cast<double *>(in), 1);
    MT_LAUNCH_CHECK();
    P->launches += 1;
    API_END
}

extern "C" mtsph_status mtsph_porous_colours(const mtsph_porous *P, int *nc) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_colours: null handle");
    *nc = P->nb.sweep == 3 ? (int)P->tiled.colour_ptr.size() - 1 : 0;
    return MTSPH_OK;
}

extern "C" mtsph_status mtsph_porous_sizes(const mtsph_porous *P, int64_t out[4]) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_sizes: null handle");
    const NbhDev &nb = P->nb;
    out[0] = nb.nnz;
    out[1] = nb.sweep == 3 ? P->tiled.npairs : nb.npairs;
    out[2] = nb.sweep == 3 ? P->tiled.npairs : nb.ngroups;
    out[3] = nb.sweep == 3 ? (int64_t)P->tiled.colour_ptr.size() - 1 : nb.sweep == 1 ? nb.nlevels : 0;
    return MTSPH_OK;
}

extern "C" mtsph_status mtsph_porous_outer_ms(const mtsph_porous *P, double *ms) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_outer_ms: null handle");
    API_BEGIN
    if (!P->ev_outer[0]) throw Error(MTSPH_ERR_ARG, "no outer step has run");
    float f = 0.f;
    MT_CUDA(cudaEventElapsedTime(&f, P->ev_outer[0], P->ev_outer[1]));
    *ms = f;
    API_END
}

extern "C" mtsph_status mtsph_porous_stable_dt(mtsph_porous *P, double cfl, double *dt) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_stable_dt: null handle");
    API_BEGIN
    P->pull_ctrl();
    P->hc->cfl = cfl;
    P->push_ctrl();
    if (P->d == 2) porous_init_dt<2>(P); else porous_init_dt<3>(P);
    P->pull_ctrl();
    *dt = P->hc->dt;
    API_END
}

extern "C" mtsph_status mtsph_porous_relax_step(mtsph_porous *P, double dt, double eta, double *ek) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_relax_step: null handle");
    API_BEGIN
    P->pull_ctrl();
    P->hc->dt = dt;
    P->hc->eta = eta;
    P->hc->done = 0;
    P->push_ctrl();
    P->launches += porous_step_any(P, CTRL_SINGLE);
    P->pull_ctrl();
    check_porous_errors(P);
    *ek = P->hc->ek;
    API_END
}

static cudaGraphExec_t porous_graph(mtsph_porous *P, int which) {
    if (P->graphs[which]) return P->graphs[which];
    cudaGraph_t g;
    MT_CUDA(cudaStreamBeginCapture(P->s, cudaStreamCaptureModeThreadLocal));
    int l = 0;
    for (int k = 0; k < P->graph_steps[which]; ++k) l = porous_step_any(P, CTRL_STEP);
    MT_CUDA(cudaStreamEndCapture(P->s, &g));
    MT_CUDA(cudaGraphInstantiate(&P->graphs[which], g, 0));
    cudaGraphDestroy(g);
    P->per_step_launches = l;
    return P->graphs[which];
}

extern "C" mtsph_status mtsph_porous_relax(mtsph_porous *P, const mtsph_inner_params *p,
                                           mtsph_inner_result *r) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_relax: null handle");
    API_BEGIN
    P->pull_ctrl();
    Ctrl *c = P->hc;
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
    c->ramp_left = 0;
    c->err_inv = c->err_rm = ~0ull;
    c->remote_err = 0;
    P->push_ctrl();
    if (P->d == 2) porous_init_dt<2>(P); else porous_init_dt<3>(P);
    int which = 0;
    while (true) {
        MT_CUDA(cudaGraphLaunch(porous_graph(P, which), P->s));
        P->launches += (int64_t)P->graph_steps[which] * P->per_step_launches;
        P->pull_ctrl();
        if (c->done) break;
        if (which < 2) ++which;
    }
    check_porous_errors(P);
    r->n_inner = c->n_inner;
    r->cap_hit = c->cap_hit;
    r->ek = c->ek;
    r->min_dt = c->min_dt;
    r->last_dt = c->last_dt;
    API_END
}

extern "C" mtsph_status mtsph_porous_refresh_velocities(mtsph_porous *P) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_refresh_velocities: null handle");
    API_BEGIN
    PorousArgs A = P->args();
    if (P->d == 2) k_por_refresh<2><<<blocks_for(P->n), 256, 0, P->s>>>(A);
    else k_por_refresh<3><<<blocks_for(P->n), 256, 0, P->s>>>(A);
    MT_LAUNCH_CHECK();
    P->launches += 1;
    MT_CUDA(cudaStreamSynchronize(P->s));
    API_END
}

static DBuf<double> *porous_field(mtsph_porous *P, const std::string &f, int &comps) {
    const int d = P->d;
    if (f == "pos") { comps = d; return &P->x; }
    if (f == "F") { comps = d * d; return &P->F; }
    if (f == "momentum") { comps = d; return &P->M; }
    if (f == "vel_fluid") { comps = d; return &P->vl; }
    if (f == "flux") { comps = d; return &P->q; }
    if (f == "fluid_mass") { comps = 1; return &P->mass_l; }
    if (f == "saturation") { comps = 1; return &P->sat; }
    if (f == "pressure") { comps = 1; return &P->pres; }
    return nullptr;
}

extern "C" mtsph_status mtsph_porous_get(mtsph_porous *P, const char *field, double *host) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_get: null handle");
    API_BEGIN
    const int64_t n = P->n;
    const int d = P->d;
    std::vector<int64_t> perm(n);
    P->nb.perm.download(perm.data(), n, P->s);
    std::string f(field);
    std::vector<double> buf;
    int comps = 0;
    if (DBuf<double> *src = porous_field(P, f, comps)) {
        buf.resize((size_t)comps * n);
        src->download(buf.data(), buf.size(), P->s);
        MT_CUDA(cudaStreamSynchronize(P->s));
        for (int64_t k = 0; k < n; ++k)
            for (int c = 0; c < comps; ++c) host[perm[k] * comps + c] = buf[(size_t)c * n + k];
    } else if (f == "vel_solid" || f == "ref_pos") {
        const int stride = (f == "ref_pos" || d == 3) ? 4 : 2;
        buf.resize((size_t)stride * n);
        const void *src = f == "vel_solid" ? (const void *)P->V.p : (const void *)P->nb.XV.p;
        MT_CUDA(cudaMemcpyAsync(buf.data(), src, buf.size() * 8, cudaMemcpyDeviceToHost, P->s));
        MT_CUDA(cudaStreamSynchronize(P->s));
        for (int64_t k = 0; k < n; ++k)
            for (int c = 0; c < d; ++c) host[perm[k] * d + c] = buf[(size_t)k * stride + c];
    } else {
        throw Error(MTSPH_ERR_ARG, "unknown porous field " + f);
    }
    API_END
}

extern "C" mtsph_status mtsph_porous_set(mtsph_porous *P, const char *field, const double *host) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_set: null handle");
    API_BEGIN
    const int64_t n = P->n;
    const int d = P->d;
    std::vector<int64_t> perm(n);
    P->nb.perm.download(perm.data(), n, P->s);
    MT_CUDA(cudaStreamSynchronize(P->s));
    std::string f(field);
    std::vector<double> buf;
    int comps = 0;
    if (DBuf<double> *dst = porous_field(P, f, comps)) {
        buf.resize((size_t)comps * n);
        for (int64_t k = 0; k < n; ++k)
            for (int c = 0; c < comps; ++c) buf[(size_t)c * n + k] = host[perm[k] * comps + c];
        dst->upload(buf.data(), buf.size(), P->s);
    } else if (f == "vel_solid") {
        const int stride = d == 3 ? 4 : 2;
        buf.assign((size_t)stride * n, 0.0);
        for (int64_t k = 0; k < n; ++k)
            for (int c = 0; c < d; ++c) buf[(size_t)k * stride + c] = host[perm[k] * d + c];
        MT_CUDA(cudaMemcpyAsync(P->V.p, buf.data(), buf.size() * 8, cudaMemcpyHostToDevice, P->s));
    } else {
        throw Error(MTSPH_ERR_ARG, "unknown or read-only porous field " + f);
    }
    MT_CUDA(cudaStreamSynchronize(P->s));
    API_END
}

extern "C" mtsph_status mtsph_porous_launches(const mtsph_porous *P, int64_t *count) {
    if (!P) return fail(MTSPH_ERR_ARG, "mtsph_porous_launches: null handle");
    *count = P->launches;
    return MTSPH_OK;
}
