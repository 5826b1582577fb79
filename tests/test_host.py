"""CPU: host-side driver logic -- config grammar, particle generation
(pinned to the reference's lattices), stepping policy and the outer/inner
driver protocol (exercised with the oracle's problem objects)."""

import numpy as np
import pytest

from conftest import rel_err

from paper_2309_04010_b200 import lattices, stepping
from paper_2309_04010_b200.config import load_config, resolve
from paper_2309_04010_b200.errors import (ConfigError, ElementInversionError,
                                          ReturnMapError, SingularMomentMatrixError)


# ---------------------------------------------------------------- config

def test_defaults_and_override(tmp_path):
    cfg = tmp_path / "a.cfg"
    cfg.write_text("scenario = necking_2d\n[stepping]\neta = 1e3  # damping\nn_outer = 1e3\n")
    c = load_config(str(cfg))
    assert c.params["eta"] == 1e3 and c.params["n_outer"] == 1000
    assert c.params["initial_flow_stress"] == 450.0e6


@pytest.mark.parametrize("text,match", [
    ("scenario = necking_2d\netta = 1\n", "unknown key 'etta'"),
    ("scenario = necking_2d\neta = 1\neta = 2\n", "duplicate key"),
    ("scenario = necking_2d\nn_outer = 2.5\n", "not a valid int"),
    ("scenario = necking_2d\ndp = -1\n", "out of range"),
    ("scenario = necking_2d\n[bogus]\n", "unknown section"),
    ("scenario = necking_2d\ndiffusivity = 1\n", "does not apply"),
    ("scenario = nope\n", "unknown scenario"),
])
def test_config_errors_name_the_problem(tmp_path, text, match):
    cfg = tmp_path / "b.cfg"
    cfg.write_text(text)
    with pytest.raises(ConfigError, match=match):
        load_config(str(cfg))


def test_every_damping_order_is_selectable_from_a_config_file(tmp_path):
    for order in ("serial", "coloured", "tiled"):
        cfg = tmp_path / f"{order}.cfg"
        cfg.write_text(f"scenario = bar_3d\ndamping_sweep = {order}\n")
        assert load_config(str(cfg)).params["damping_sweep"] == order


@pytest.mark.parametrize("raw,match", [
    ({"dp": -0.1}, "out of range"),
    ({"damping_sweep": "random"}, "invalid"),
    ({"n_outer": 2.5}, "not a valid int"),
    ({"eta": "fast"}, "not a valid float"),
    ({"h_factor": 0.0}, "out of range"),
])
def test_dict_input_and_overrides_are_validated_like_files(raw, match):
    with pytest.raises(ConfigError, match=match):
        resolve({"scenario": "bar_2d", **raw})
    key, value = next(iter(raw.items()))
    with pytest.raises(ConfigError, match=match):
        resolve({"scenario": "bar_2d"}, overrides={key: value})


def test_fsi_auto_outer_steps():
    p = resolve({"scenario": "fsi_3d", "dp": 0.125e-3 / 2}).params
    h = p["h_factor"] * p["dp"]
    assert p["n_outer"] == int(np.ceil(p["t_total"] / (0.5 * h * h / p["diffusivity"])))


def test_baseline_workloads():
    p = resolve({"scenario": "bar_3d"}).params
    assert lattices.particle_count(p) == 1000 * 100 * 100
    c = np.sqrt(p["bulk_modulus"] / p["density"])
    assert p["eta"] == pytest.approx(0.1 * c * 1.3 * 0.02)
    assert p["cfl"] == 0.2 and p["hardening_law"] == "power"
    assert lattices.particle_count(resolve({"scenario": "bar_2d"}).params) == 4000
    assert lattices.particle_count(resolve({"scenario": "membrane_2d"}).params) == (400 + 4) * 20


# ---------------------------------------------------------------- lattices

@pytest.mark.parametrize("prefix,raw", [
    ("n2_", {"scenario": "necking_2d", "length": 8e-3, "width": 2e-3, "dp": 0.25e-3}),
    ("n3_", {"scenario": "necking_3d", "length": 8e-3, "radius": 2e-3, "dp": 0.5e-3}),
])
def test_necking_lattices_match_reference(gold_traj, prefix, raw):
    raw = dict(raw, n_outer=4)
    lat = lattices.build_lattice(resolve(raw).params)
    np.testing.assert_array_equal(lat.pos, gold_traj[prefix + "ref_pos"])
    np.testing.assert_array_equal(lat.vol, gold_traj[prefix + "vol"])
    np.testing.assert_array_equal(lat.constrained, gold_traj[prefix + "constrained"])


@pytest.mark.parametrize("prefix,raw", [
    ("nbhfsi2d_", {"scenario": "fsi_2d", "length": 2e-3}),
    ("nbhneck3d_", {"scenario": "necking_3d", "length": 8e-3, "radius": 2e-3, "dp": 0.5e-3,
                    "n_outer": 4}),
    ("nbhfsi3d_", {"scenario": "fsi_3d", "length": 0.5e-3, "breadth": 0.5e-3,
                   "dp": 0.125e-3 / 4}),
])
def test_scenario_lattices_and_kernels_match_reference(gold_nbh, prefix, raw):
    lat = lattices.build_lattice(resolve(raw).params)
    np.testing.assert_array_equal(lat.pos, gold_nbh[prefix + "pos"])
    np.testing.assert_array_equal(lat.vol, gold_nbh[prefix + "vol"])
    h_axes = float(gold_nbh[prefix + "h"]) * gold_nbh[prefix + "aniso"]
    np.testing.assert_array_equal(lat.h_axes, h_axes)


def test_paper_particle_counts():
    assert abs(lattices.particle_count(resolve({"scenario": "necking_2d"}).params) - 10788) \
        <= 0.05 * 10788
    assert abs(lattices.particle_count(resolve({"scenario": "necking_3d"}).params) - 250852) \
        <= 0.05 * 250852
    assert lattices.particle_count(resolve({"scenario": "fsi_2d"}).params) == 1336
    assert lattices.particle_count(resolve({"scenario": "fsi_3d"}).params) == 60552


def test_bad_spacing_and_coarse_cylinder_rejected():
    with pytest.raises(ConfigError, match="0.5%"):
        lattices.build_lattice(resolve({"scenario": "necking_2d", "dp": 1.9e-3, "n_outer": 10}).params)
    with pytest.raises(ConfigError, match="diameter"):
        lattices.build_lattice(resolve({"scenario": "necking_3d", "dp": 53.334e-3 / 20,
                                        "n_outer": 10}).params)


def test_fsi_contact_and_clamps():
    lat = lattices.build_lattice(resolve({"scenario": "fsi_2d"}).params)
    assert lat.contact.sum() == 49 * 4
    assert lat.constrained.sum() == 6 * 8


def test_jittered_block_is_seeded():
    a = lattices.build_lattice(resolve({"scenario": "block_3d", "length": 0.2, "width": 0.1,
                                        "breadth": 0.1, "seed": 3}).params)
    b = lattices.build_lattice(resolve({"scenario": "block_3d", "length": 0.2, "width": 0.1,
                                        "breadth": 0.1, "seed": 3}).params)
    np.testing.assert_array_equal(a.pos, b.pos)
    c = lattices.build_lattice(resolve({"scenario": "block_3d", "length": 0.2, "width": 0.1,
                                        "breadth": 0.1, "jitter": 0.0}).params)
    dev = np.max(np.abs(a.pos - c.pos))
    assert 0.02 * 0.04 < dev <= 0.05 * 0.02 + 1e-15


# ---------------------------------------------------------------- stepping

def test_policy_and_time_steps():
    pol = stepping.SteppingPolicy(dt_outer=1.0, n_outer=1, eta=0.0, energy_criterion=1.0,
                                  energy_reference=1.0)
    assert pol.inner_cap(1e-3) == 10000
    with pytest.raises(ValueError):
        stepping.SteppingPolicy(dt_outer=1.0, n_outer=1, eta=0.0, energy_criterion=1.0,
                                energy_reference=1.0, energy_mode="bogus")
    assert stepping.diffusion_time_step(2.03e-5, 1e-10) == pytest.approx(2.06, abs=0.01)
    rep = stepping.kinetic_energy(np.array([[2.0, 0.0], [0.0, 1.0]]), np.array([1.0, 4.0]),
                                  np.ones(2, bool), 1.0, 10.0)
    assert rep.value == pytest.approx(4.0) and rep.ratio == pytest.approx(0.4)


class _OracleAdapter:
    """Reference-protocol wrapper around the oracle necking problem."""

    def __init__(self, prob):
        self.p = prob

    ramp_active = property(lambda self: self.p.ramp_active)

    def advance_slow(self, step, dt, t):
        return self.p.advance_slow(step, dt, t)

    def stable_time_step(self, cfl):
        return self.p.stable_time_step(cfl)

    def relax_step(self, dt, eta):
        self.p.relax_step(dt, eta)

    def energy_report(self, policy):
        v = self.p.ek_pre
        return stepping.EnergyReport(v, policy.energy_reference, policy.energy_criterion,
                                     v <= policy.energy_criterion)

    def measure(self, t):
        return self.p.measure(t)

    def velocities(self):
        return self.p.vel


def test_driver_protocol_matches_reference_run(gold_runs):
    """run_outer_inner (host driver) over a reference-protocol problem."""
    from oracle.problems import NeckingOracle
    p = resolve({"scenario": "necking_2d", "length": 8e-3, "width": 2e-3, "dp": 0.5e-3,
                 "stretch_per_end": 4e-6, "n_outer": 4, "ramp_steps": 3, "eta": 1e4,
                 "energy_pct": 0.005, "energy_ref": 1e-4}).params
    lat = lattices.build_lattice(p)
    prob = _OracleAdapter(NeckingOracle(
        lat.pos, lat.vol, 7850.0, lat.constrained, lat.side < 0, lat.side > 0, lat.mid_mask,
        80.1938e9, 164.21e9, (450e6, 715e6, 16.93, 129.24e6), 1.35 * 0.5e-3,
        end_disp_per_outer=1e-6, ramp_steps=3))
    from paper_2309_04010_b200.scenarios import make_policy
    obs, counters = stepping.run_outer_inner(prob, make_policy(p, 1.35 * 0.5e-3))
    np.testing.assert_array_equal(obs.n_inner, gold_runs["rn2_n_inner"])
    np.testing.assert_allclose(obs.reaction_force, gold_runs["rn2_reaction_force"], rtol=1e-9)
    assert counters.n_damping == counters.n_inner and not counters.cap_hits
    assert rel_err(prob.p.pos, gold_runs["rn2_pos"]) < 1e-10


def test_error_messages_match_reference_format():
    assert str(ElementInversionError([3, 1])) == \
        "non-positive deformation determinant at 2 particle(s), first ids: [3, 1]"
    e = SingularMomentMatrixError([0, 1, 2, 3, 4], [0.0] * 5)
    assert e.particle_ids == [0, 1, 2, 3, 4] and "first ids: [0, 1, 2, 3, 4]" in str(e)
    assert ReturnMapError([7], [1.0]).residuals == [1.0]
