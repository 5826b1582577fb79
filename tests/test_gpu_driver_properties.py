"""GPU: the reference's driver-level property tests, restated against this
package's drop-in driver API (scenarios.build + stepping.run_outer_inner,
whose inner loops run on the device).  Each test names the reference test
whose property it checks (files under /root/reference/pkg/tests); the
problems are the reference's own small ("desk") configurations.
"""

import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _build(**over):
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import build
    return build(resolve(over).params)


def _desk(**over):
    """test_stepping.py:146 desk problem (2D necking bar, 16 x 4 particles)."""
    base = {"scenario": "necking_2d", "length": 8e-3, "width": 2e-3, "dp": 0.5e-3,
            "stretch_per_end": 4e-6, "n_outer": 4, "ramp_steps": 3, "eta": 1e4,
            "energy_pct": 0.005, "energy_ref": 1e-4}
    base.update(over)
    return _build(**base)


def test_zero_load_exits_at_min_inner():
    """test_stepping.py:153: no loading -> every inner loop stops at min_inner
    with the energy ratio under the criterion."""
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = _desk(stretch_per_end=1e-30, min_inner=2)
    problem.end_disp_per_outer = 0.0
    obs, counters = run_outer_inner(problem, policy)
    assert counters.n_outer == 4
    assert np.all(obs.n_inner == 2)
    assert np.all(obs.ek_ratio <= policy.energy_criterion / policy.energy_reference)


def test_damping_counter_equals_inner():
    """test_stepping.py:161: one damping sweep per inner step."""
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = _desk()
    obs, counters = run_outer_inner(problem, policy)
    assert counters.n_damping == counters.n_inner > 0
    np.testing.assert_array_equal(obs.ns_cum, obs.nd_cum)
    assert counters.n_inner == int(obs.ns_cum[-1])


def test_cap_hit_recorded_not_silent():
    """test_stepping.py:168: an inner loop stopped by max_inner is reported."""
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = _desk(max_inner=4, ramp_steps=3)
    obs, counters = run_outer_inner(problem, policy)
    assert len(counters.cap_hits) > 0 and counters.warnings
    assert np.all(obs.n_inner <= 4)


def test_converged_loops_satisfy_criterion_and_time_increases():
    """test_stepping.py:174 and :181: every loop ends under the criterion;
    the observation times increase strictly."""
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = _desk(n_outer=6)
    obs, counters = run_outer_inner(problem, policy)
    assert not counters.cap_hits
    assert np.all(obs.ek_ratio <= policy.energy_criterion / policy.energy_reference + 1e-15)
    assert np.all(np.diff(obs.time) > 0)


def test_plastic_state_alpha_monotone_and_isochoric():
    """test_plasticity.py:184 / :192 on the device state of a pulled bar:
    the equivalent plastic strain never decreases from one outer step to the
    next, and det of the stored inverse plastic tensor stays at 1."""
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = _desk(stretch_per_end=2e-4, n_outer=5)
    alphas = []
    run_outer_inner(problem, policy,
                    observers=[lambda step, t, s: alphas.append(problem.plastic.alpha)])
    assert np.max(alphas[-1]) > 0, "the bar must yield"
    for a0, a1 in zip(alphas, alphas[1:]):
        assert np.all(a1 >= a0)
    cp = problem.plastic.cp_inv
    np.testing.assert_allclose(np.linalg.det(cp), 1.0, rtol=0, atol=1e-8)


def test_load_release_returns_home():
    """test_scenarios.py:183: stretch an elastic bar, pull it back, settle:
    the residual displacement vanishes."""
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = _build(scenario="necking_2d", length=8e-3, width=2e-3, dp=0.25e-3,
                             imperfection=0.0, plasticity=False, n_outer=4,
                             stretch_per_end=2.0e-6, t_total=1.0, ramp_steps=20,
                             energy_ref=1.0, energy_pct=1e-16)
    run_outer_inner(problem, policy)
    peak = np.max(np.abs(problem.state.pos - problem.state.ref_pos))
    assert peak > 1.5e-6
    problem.end_disp_per_outer = -problem.end_disp_per_outer
    run_outer_inner(problem, policy)
    problem.end_disp_per_outer = 0.0
    run_outer_inner(problem, dataclasses.replace(policy, n_outer=2))
    final = np.max(np.abs(problem.state.pos - problem.state.ref_pos))
    assert final <= 1e-4 * peak


@pytest.mark.parametrize("sweep", ["serial", "tiled"])
def test_uniform_state_stays_exactly_at_rest(sweep):
    """test_scenarios.py:208: a membrane with no saturation gradient and no
    pressure does not move, exactly (both damping orders)."""
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import build
    from paper_2309_04010_b200.stepping import run_outer_inner
    p = resolve({"scenario": "fsi_2d", "length": 2e-3, "t_total": 4.0, "n_outer": 4,
                 "contact_time": 1e-6, "max_inner": 3, "min_inner": 1}).params
    problem, policy = build(p, sweep=sweep)
    ref = problem.state.ref_pos.copy()
    run_outer_inner(problem, policy)
    np.testing.assert_array_equal(problem.state.pos, ref)
    np.testing.assert_array_equal(problem.state.vel_solid, 0.0)
    np.testing.assert_array_equal(problem.state.flux, 0.0)
    np.testing.assert_array_equal(problem.state.pressure, 0.0)


@pytest.mark.parametrize("sweep", ["serial", "tiled"])
def test_solid_at_rest_stays_exactly_at_rest(sweep):
    """The solid counterpart: an unloaded elastoplastic bar keeps x = X,
    v = 0, F = I and alpha = 0 bit for bit through device inner steps."""
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import build
    p = resolve({"scenario": "necking_2d", "length": 8e-3, "width": 2e-3, "dp": 0.5e-3}).params
    problem, policy = build(p, sweep=sweep)
    dev, lat = problem.dev, problem.lattice
    d = lat.pos.shape[1]
    for _ in range(20):
        dev.relax_step(dev.stable_dt(policy.cfl), policy.eta)
    np.testing.assert_array_equal(dev.get("pos"), lat.pos)
    np.testing.assert_array_equal(dev.get("vel"), 0.0)
    np.testing.assert_array_equal(dev.get("F"), np.broadcast_to(np.eye(d), (lat.n, d, d)))
    np.testing.assert_array_equal(dev.get("alpha"), 0.0)


def test_porous_outer_step_conserves_fluid_mass():
    """test_porous.py:116 on the device outer step: with no wetted face and
    no evaporation the pairwise flux moves water between particles only, so
    the total fluid mass is conserved to rounding over 20 outer steps."""
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.device import DevicePorous
    from paper_2309_04010_b200.scenarios import _membrane, make_policy
    p = resolve({"scenario": "fsi_2d", "length": 2e-3}).params
    lat = lattices.build_lattice(p)
    model = _membrane(p)
    dev = DevicePorous(lat.pos, lat.vol, lat.constrained, np.zeros(lat.n, bool), lat.h_axes,
                       model, p["contact_time"], 0.0)
    rng = np.random.default_rng(3)
    m0 = rng.uniform(0.05, 0.35, lat.n) * model.fluid_density0 * lat.vol
    dev.set("fluid_mass", m0)
    dt = make_policy(p, float(np.min(lat.h_axes))).dt_outer
    clamped = 0
    for k in range(20):
        clamped += dev.advance_slow(dt, (k + 1) * dt)
    m1 = dev.get("fluid_mass")
    assert clamped == 0
    assert np.max(np.abs(m1 - m0)) > 0, "water must move"
    assert np.sum(m1) == pytest.approx(np.sum(m0), rel=1e-12)
