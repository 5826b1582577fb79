"""CPU: the oracle is pinned to the reference's own outputs (golden
fixtures written by tests/golden/make_golden.py from the real reference).

Bars: neighbour structure (CSR, pair order, damping groups) bit-exact;
damping sweep bit-exact; operators / stresses within 1e-14 of the field
scale; per-step trajectories within 1e-10 over 100 inner steps.
"""

import numpy as np
import pytest

from conftest import rel_err

from oracle import oracle as O
from oracle.problems import NeckingOracle, PorousOracle, run_outer_inner

NBH = ["nbh2d_", "nbh3d_", "nbh2d13_", "nbhfsi2d_", "nbhneck3d_", "nbhfsi3d_"]


def _g(data, prefix):
    return {k[len(prefix):]: data[k] for k in data.files if k.startswith(prefix)}


@pytest.mark.parametrize("case", NBH)
def test_neighbourhood_bit_exact(gold_nbh, case):
    g = _g(gold_nbh, case)
    nb = O.build_nbh(g["pos"], g["vol"], float(g["h"]), g["aniso"])
    for k in ("indptr", "idx", "pair_i", "pair_j", "pair_group"):
        np.testing.assert_array_equal(getattr(nb, k), g[k])
    np.testing.assert_array_equal(nb.grad0, g["grad0"])
    np.testing.assert_array_equal(nb.pair_damp, g["pair_damp"])
    assert rel_err(nb.corr, g["corr"]) < 1e-14


@pytest.mark.parametrize("op,nb", [("op2d_", "nbh2d_"), ("op3d_", "nbh3d_")])
def test_operators(gold_ops, gold_nbh, op, nb):
    g = _g(gold_nbh, nb)
    o = _g(gold_ops, op)
    nbh = O.build_nbh(o["pos"], o["vol"], 1.35)
    assert rel_err(O.deformation_rate(o["vel"], nbh), o["rate"]) < 1e-14
    assert rel_err(O.stress_divergence(o["pk1"], 7850.0, nbh), o["acc"]) < 1e-14
    out = O.damping_sweep(o["damp_vin"].copy(), o["mass"], o["movable"], nbh, 1e3, 1e-3)
    np.testing.assert_array_equal(out, o["damp_vout"])
    assert g["pos"].shape == o["pos"].shape


@pytest.mark.parametrize("nb", ["nbhfsi2d_", "nbhneck3d_", "nbhfsi3d_"])
def test_damping_groups_bit_exact(gold_nbh, gold_ops, nb):
    g = _g(gold_nbh, nb)
    k = "damp_" + nb
    nbh = O.build_nbh(g["pos"], g["vol"], float(g["h"]), g["aniso"])
    assert np.max(np.diff(nbh.pair_group)) > 1, "case must contain multi-pair groups"
    out = O.damping_sweep(gold_ops[k + "vin"].copy(), gold_ops[k + "mass"],
                          gold_ops[k + "movable"], nbh, float(gold_ops[k + "eta"]),
                          float(gold_ops[k + "dt"]))
    np.testing.assert_array_equal(out, gold_ops[k + "vout"])


@pytest.mark.parametrize("d", [3, 2])
def test_return_map(gold_const, d):
    c = gold_const
    mu, K, _ = c["steel"]
    p = f"rm{d}d_"
    matp = O.material_vector(mu, K, *c["hard"])
    tau, pk1, cp, al, pl, dg = O.return_map(c[p + "F"], c[p + "cp"], c[p + "alpha"], matp)
    np.testing.assert_array_equal(pl, c[p + "plastic"])
    assert rel_err(tau, c[p + "tau"]) < 1e-14
    assert rel_err(pk1, c[p + "pk1"]) < 1e-14
    assert rel_err(cp, c[p + "cp_new"]) < 1e-14
    assert rel_err(al, c[p + "alpha_new"]) < 1e-14
    assert rel_err(dg, c[p + "dgamma"]) < 1e-13
    tau_el, pk1_el, *_ = O.return_map(c[p + "F"], c[p + "cp"], c[p + "alpha"], matp,
                                      elastic_only=True)
    assert rel_err(tau_el, c[p + "tau_el"]) < 1e-14


@pytest.mark.parametrize("p", ["p2d_", "p3d_"])
def test_porous_kernels(gold_porous, p):
    gp = gold_porous
    m = O.Membrane(*gp["model"])
    nbh = O.build_nbh(gp[p + "pos"], gp[p + "vol"], 1.35e-5)
    F, vol = gp[p + "F"], gp[p + "vol"]
    sat, q = O.saturation_and_flux(F, gp[p + "mass_in"], vol, nbh, m)
    assert rel_err(sat, gp[p + "sat"]) < 1e-14
    assert rel_err(q, gp[p + "q"]) < 1e-14
    mass, cl = O.fluid_mass_update(F, gp[p + "mass_in"], gp[p + "flux_in"], vol, nbh, m, 50.0)
    assert rel_err(mass, gp[p + "mass_out"]) < 1e-14 and cl == int(gp[p + "clamped"])
    tb, j, rate, bad = O.porous_stress_rhs(F, gp[p + "pressure"], nbh, m)
    assert bad == 0 and rel_err(tb, gp[p + "tbuf"]) < 1e-14
    assert rel_err(rate, gp[p + "stress_rate"]) < 1e-14
    fr = O.momentum_flux_rate(F, gp[p + "vel_fluid"], gp[p + "flux_in"], vol, nbh)
    assert rel_err(fr, gp[p + "flux_rate"]) < 1e-14
    vs, vl = O.split_velocities(F, gp[p + "mass_in"], gp[p + "momentum"], gp[p + "flux_in"],
                                vol, m)
    assert rel_err(vs, gp[p + "v_s"]) < 1e-14 and rel_err(vl, gp[p + "v_l"]) < 1e-14


@pytest.mark.parametrize("prefix", ["n2_", "n3_"])
def test_necking_trajectory(gold_traj, prefix):
    pos = gold_traj[prefix + "ref_pos"]
    con = gold_traj[prefix + "constrained"]
    d = pos.shape[1]
    dp = 0.25e-3 if d == 2 else 0.5e-3
    prob = NeckingOracle(pos, gold_traj[prefix + "vol"], 7850.0, con, con & (pos[:, 0] < 0),
                         con & (pos[:, 0] > 0), np.abs(pos[:, 0]) <= 0.51 * dp, 80.1938e9,
                         164.21e9, (450e6, 715e6, 16.93, 129.24e6), 1.35 * dp,
                         end_disp_per_outer=3e-5, ramp_steps=20)
    prob.advance_slow(1, 25.0, 25.0)
    for k in range(1, 101):
        dt = prob.stable_time_step(0.6)
        assert abs(dt - gold_traj[prefix + "dt"][k - 1]) <= 1e-12 * dt
        prob.relax_step(dt, 1e4)
        if k in (1, 10, 50, 100):
            s = f"{prefix}s{k}_"
            for ours, key in ((prob.pos, "pos"), (prob.vel, "vel"), (prob.F, "F"),
                              (prob.alpha, "alpha"), (prob.cp, "cp"), (prob.accel, "accel")):
                assert rel_err(ours, gold_traj[s + key]) < 1e-10, (k, key)


def test_necking_run_observables(gold_runs):
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    p = resolve({"scenario": "necking_2d", "length": 8e-3, "width": 2e-3, "dp": 0.5e-3,
                 "stretch_per_end": 4e-6, "n_outer": 4, "ramp_steps": 3, "eta": 1e4,
                 "energy_pct": 0.005, "energy_ref": 1e-4}).params
    lat = lattices.build_lattice(p)
    prob = NeckingOracle(lat.pos, lat.vol, 7850.0, lat.constrained, lat.side < 0, lat.side > 0,
                         lat.mid_mask, 80.1938e9, 164.21e9, (450e6, 715e6, 16.93, 129.24e6),
                         1.35 * 0.5e-3, end_disp_per_outer=1e-6, ramp_steps=3)
    rows = run_outer_inner(prob, 25.0, 4, 1e4, 0.005 * 1e-4)
    np.testing.assert_array_equal([r["n_inner"] for r in rows], gold_runs["rn2_n_inner"])
    np.testing.assert_allclose([r["reaction_force"] for r in rows],
                               gold_runs["rn2_reaction_force"], rtol=1e-9)
    assert rel_err(prob.pos, gold_runs["rn2_pos"]) < 1e-10


def test_porous_run_observables(gold_runs):
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    p = resolve({"scenario": "fsi_2d", "length": 2e-3, "t_total": 2.4, "n_outer": 3,
                 "contact_time": 0.8, "max_inner": 40}).params
    lat = lattices.build_lattice(p)
    m = O.Membrane(p["density"], p["diffusivity"], p["pressure_coeff"], p["youngs_modulus"],
                   p["poisson_ratio"], p["porosity"], p["fluid_density"], p["initial_saturation"])
    prob = PorousOracle(lat.pos, lat.vol, lat.constrained, lat.contact, m, p["h_factor"] * p["dp"],
                        (p["anisotropy"], 1.0), p["contact_time"], p["evaporation_rate"],
                        lat.column_id, len(lat.column_x), lat.center_column, lat.deflection_axis)
    ref = p["pressure_coeff"] * (p["porosity"] - p["initial_saturation"])
    rows = run_outer_inner(prob, 0.8, 3, p["eta"], p["energy_pct"] * ref, max_inner=40)
    np.testing.assert_array_equal([r["n_inner"] for r in rows], gold_runs["rf2_n_inner"])
    assert rel_err(prob.fluid_mass, gold_runs["rf2_fluid_mass"]) < 1e-10
    assert rel_err(prob.pos - lat.pos, gold_runs["rf2_pos"] - lat.pos) < 1e-8
    assert rel_err(np.array([r["profile"] for r in rows]), gold_runs["rf2_profile"]) < 1e-8


def test_desk_necking_acceptance_head():
    """The oracle against the reference's own run of its acceptance
    configuration (desk necking bar, dp = PH/25; tests/golden/
    acceptance_heads.npz): 12 outer steps through first mid-span yield."""
    from conftest import golden
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import _necking_materials, make_policy
    gold = golden("acceptance_heads.npz")
    p = resolve({"scenario": "necking_2d", "dp": 12.826e-3 / 25, "n_outer": 1000}).params
    lat = lattices.build_lattice(p)
    el, hard = _necking_materials(p)
    law, hp = hard.device_params()
    policy = make_policy(p, float(np.min(lat.h_axes)))
    prob = NeckingOracle(lat.pos, lat.vol, el.density0, lat.constrained, lat.side < 0,
                         lat.side > 0, lat.mid_mask, el.shear_modulus, el.bulk_modulus, hp,
                         float(lat.h_axes[0]), end_disp_per_outer=p["stretch_per_end"] / p["n_outer"],
                         ramp_steps=p["ramp_steps"], hardening_law=law)
    n_outer = len(gold["an2_n_inner"])
    rows = run_outer_inner(prob, policy.dt_outer, n_outer, policy.eta, policy.energy_criterion,
                           cfl=policy.cfl, max_inner=policy.max_inner, min_inner=policy.min_inner)
    np.testing.assert_array_equal([r["n_inner"] for r in rows], gold["an2_n_inner"])
    for key in ("reaction_force", "mid_alpha_min"):
        got = np.array([r[key] for r in rows])
        assert rel_err(got, gold["an2_" + key]) < 1e-9, key
    assert np.max(gold["an2_mid_alpha_min"]) > 0
    assert rel_err(prob.pos - lat.pos, gold["an2_pos"] - lat.pos) < 1e-9
