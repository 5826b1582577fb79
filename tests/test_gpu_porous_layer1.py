"""GPU parity: _accel.py drop-ins (layer 1) and the porous membrane problem.

Layer-1 entry points take the reference's own arrays (golden
neighbourhoods) and must reproduce the reference outputs to round-off
(1e-13 relative to the field scale; the damping sweep to 1e-14).  The
device-resident porous problem must reproduce whole reference runs
(fsi_2d / fsi_3d, serial damping order) to 1e-9 in positions and fluid
masses.
"""

import ctypes

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2309_04010_b200 import _lib
    return _lib.load_library(), _lib.ptr, _lib.check


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


@pytest.mark.parametrize("op,nb", [("op2d_", "nbh2d_"), ("op3d_", "nbh3d_")])
def test_layer1_gathers_match_reference(gold_nbh, gold_ops, op, nb):
    lib, ptr, check = _lib()
    g = {k[len(nb):]: gold_nbh[k] for k in gold_nbh.files if k.startswith(nb)}
    n, d = g["pos"].shape
    ip, idx, grad, vol = _c(g["indptr"], np.int64), _c(g["idx"], np.int64), _c(g["grad0"]), _c(g["vol"])
    raw = np.zeros((n, d, d))
    check(lib.mtsph_velocity_gradient_gather(n, d, ptr(_c(gold_ops[op + "vel"])), ptr(ip), ptr(idx),
                                             ptr(grad), ptr(vol), ptr(raw)))
    assert rel_err(raw @ g["corr"], gold_ops[op + "rate"]) < 1e-13
    t = _c(gold_ops[op + "pk1"] @ g["corr"])
    acc = np.zeros((n, d))
    check(lib.mtsph_pair_tensor_divergence(n, d, ptr(t), ptr(ip), ptr(idx), ptr(grad), ptr(vol), ptr(acc)))
    assert rel_err(acc / 7850.0, gold_ops[op + "acc"]) < 1e-13


def _sweep(lib, ptr, check, vel, mass, movable, g, eta, dt):
    n, d = vel.shape
    inv = np.where(movable, 1.0 / mass, 0.0)
    pi, pj = _c(g["pair_i"], np.int64), _c(g["pair_j"], np.int64)
    v = _c(vel).copy()
    check(lib.mtsph_damping_sweep(n, d, ptr(v), len(pi), ptr(pi), ptr(pj), ptr(_c(g["pair_damp"])),
                                  ptr(_c(inv[pi])), ptr(_c(inv[pj])), len(g["pair_group"]) - 1,
                                  ptr(_c(g["pair_group"], np.int64)), eta, dt))
    return v


@pytest.mark.parametrize("nb", ["nbh2d_", "nbh3d_", "nbhfsi2d_", "nbhneck3d_", "nbhfsi3d_"])
def test_layer1_damping_sweep_matches_reference(gold_nbh, gold_ops, nb):
    lib, ptr, check = _lib()
    g = {k[len(nb):]: gold_nbh[k] for k in gold_nbh.files if k.startswith(nb)}
    if nb in ("nbh2d_", "nbh3d_"):
        op = "op2d_" if nb == "nbh2d_" else "op3d_"
        args = (gold_ops[op + "damp_vin"], gold_ops[op + "mass"], gold_ops[op + "movable"], 1e3, 1e-3)
        want = gold_ops[op + "damp_vout"]
    else:
        k = "damp_" + nb
        args = (gold_ops[k + "vin"], gold_ops[k + "mass"], gold_ops[k + "movable"],
                float(gold_ops[k + "eta"]), float(gold_ops[k + "dt"]))
        want = gold_ops[k + "vout"]
    vel, mass, movable, eta, dt = args
    out = _sweep(lib, ptr, check, vel, mass, movable, g, eta, dt)
    assert rel_err(out, want) < 1e-14


@pytest.mark.parametrize("p", ["p2d_", "p3d_"])
def test_layer1_porous_kernels_match_reference(gold_porous, p):
    """porous.py:141/168/239 and _accel.py:240 through the drop-ins."""
    from oracle import oracle as O
    lib, ptr, check = _lib()
    gp = gold_porous
    pos, vol = gp[p + "pos"], gp[p + "vol"]
    n, d = pos.shape
    nbh = O.build_nbh(pos, vol, 1.35e-5)   # structure already pinned bit-exact
    F = _c(gp[p + "F"])
    m = O.Membrane(*gp["model"])
    j = np.linalg.det(F)
    volc = _c(vol * j)
    amap = _c(np.linalg.inv(F) @ np.swapaxes(nbh.corr, -1, -2))
    rho_l = gp[p + "mass_in"] / volc
    sat = _c(rho_l / m.fluid_density0)
    coeff = _c(m.diffusivity * rho_l)
    q = np.zeros((n, d))
    check(lib.mtsph_scalar_difference_flux(n, d, ptr(sat), ptr(coeff), ptr(amap), ptr(nbh.indptr),
                                           ptr(nbh.idx), ptr(volc), ptr(nbh.grad0), ptr(q)))
    assert rel_err(q, gp[p + "q"]) < 1e-13
    rate = np.zeros(n)
    check(lib.mtsph_conservative_mass_rate(n, d, ptr(_c(gp[p + "flux_in"])), ptr(amap), len(nbh.pair_i),
                                           ptr(nbh.pair_i), ptr(nbh.pair_j), ptr(nbh.pair_grad),
                                           ptr(volc), ptr(rate)))
    mass = np.clip(gp[p + "mass_in"] + 50.0 * rate, 0.0, m.porosity * m.fluid_density0 * volc)
    assert rel_err(mass, gp[p + "mass_out"]) < 1e-13
    tbuf = np.zeros((n, d, d))
    jout = np.zeros(n)
    srate = np.zeros((n, d))
    check(lib.mtsph_porous_stress_rhs(n, d, ptr(F), ptr(_c(gp[p + "pressure"])), ptr(nbh.corr),
                                      ptr(nbh.indptr), ptr(nbh.idx), ptr(nbh.grad0), ptr(_c(vol)),
                                      m.mu, m.lam, ptr(tbuf), ptr(jout), ptr(srate)))
    assert rel_err(tbuf, gp[p + "tbuf"]) < 1e-13
    assert rel_err(srate, gp[p + "stress_rate"]) < 1e-13
    vq = _c(gp[p + "vel_fluid"][:, :, None] * gp[p + "flux_in"][:, None, :])
    frate = np.zeros((n, d))
    check(lib.mtsph_pair_tensor_divergence_mapped(n, d, ptr(vq), ptr(_c(-amap)), ptr(nbh.indptr),
                                                  ptr(nbh.idx), ptr(nbh.grad0), ptr(volc), ptr(frate)))
    assert rel_err(frate, gp[p + "flux_rate"]) < 1e-13


FSI_RUNS = {
    "rf2_": {"scenario": "fsi_2d", "length": 2e-3, "t_total": 2.4, "n_outer": 3,
             "contact_time": 0.8, "max_inner": 40},
    "rf3_": {"scenario": "fsi_3d", "length": 0.5e-3, "breadth": 0.5e-3, "dp": 0.125e-3 / 4,
             "t_total": 3.0, "n_outer": 3, "contact_time": 1.0, "max_inner": 30, "min_inner": 5},
}


@pytest.mark.parametrize("prefix", sorted(FSI_RUNS))
def test_porous_run_matches_reference(gold_runs, prefix):
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = scenarios.build(resolve(FSI_RUNS[prefix]).params, sweep="serial")
    obs, counters = run_outer_inner(problem, policy)
    g = gold_runs
    np.testing.assert_array_equal(obs.n_inner, g[prefix + "n_inner"])
    assert counters.clamp_events == int(g[prefix + "clamp"])
    st = problem.state
    assert rel_err(st.pos - st.ref_pos, g[prefix + "pos"] - st.ref_pos) < 1e-8
    assert rel_err(st.fluid_mass, g[prefix + "fluid_mass"]) < 1e-10
    assert rel_err(st.saturation, g[prefix + "saturation"]) < 1e-10
    assert rel_err(st.vel_solid, g[prefix + "vel"]) < 1e-7
    assert rel_err(obs.extras["profile"], g[prefix + "profile"]) < 1e-8
    assert rel_err(obs.amplitude, g[prefix + "amplitude"]) < 1e-8
