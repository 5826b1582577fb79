"""GPU parity on the BASELINE.json workloads themselves (the configs that are
parity cases, not bench lines), against the CPU oracle on the same inputs:

  configs[0] bar_2d: 2D plane-strain power-law-hardening bar 20 x 2,
             dp 0.1 (4000 particles), right end pulled -- 100 inner steps
             with the stretch ramp active, every field <= 1e-10 (north-star
             per-step bar), serial (reference) damping order;
  configs[1] membrane_2d: 2D strip 10 x 0.5, dp 0.025 (8000 + clamp
             particles), saturation held on the top face, swelling through
             the pore-pressure law -- three outer diffusion steps with
             their inner relaxations, fluid mass / saturation <= 1e-10,
             displacement <= 1e-8 (the reference-run tolerances of
             test_gpu_porous_layer1.py);
  configs[3] membrane_3d: the same material and wetting on the 3D cantilever
             plate (40 x 40 x 1 at dp 1/22 in the bench; a 1 x 0.5 x 1 piece
             of it here, 6292 particles) -- the same three-outer-step run.
"""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


def test_config0_bar2d_trajectory_matches_oracle():
    from oracle.problems import NeckingOracle
    from paper_2309_04010_b200 import device, lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import _necking_materials
    p = resolve({"scenario": "bar_2d"}).params
    lat = lattices.build_lattice(p)
    assert lat.n == 4000
    el, hard = _necking_materials(p)
    law, hp = hard.device_params()
    assert law == 1                                   # BASELINE power law
    gpu = device.DeviceSolid(lat.pos, lat.vol, el.density0, lat.constrained, lat.side,
                             lat.mid_mask, lat.h_axes, el.shear_modulus, el.bulk_modulus,
                             plastic=True, hardening_law=law, hard=hp, sweep="serial")
    # a faster pull than the BASELINE's 1e-3 per unit time so 100 steps
    # reach plastic flow at the pulled ends: 0.2 % of the length per end
    disp, ramp = 0.002 * p["length"], 100
    cpu = NeckingOracle(lat.pos, lat.vol, el.density0, lat.constrained, lat.side < 0,
                        lat.side > 0, lat.mid_mask, el.shear_modulus, el.bulk_modulus, hp,
                        float(lat.h_axes[0]), end_disp_per_outer=disp, ramp_steps=ramp,
                        hardening_law=law)
    gpu.set_ramp(disp, ramp, ramp)
    cpu.advance_slow(1, 1.0, 1.0)
    cfl, eta = p["cfl"], p["eta"]
    for _ in range(100):
        dt = gpu.stable_dt(cfl)
        dtc = cpu.stable_time_step(cfl)
        assert abs(dt - dtc) <= 1e-10 * dtc
        gpu.relax_step(dt, eta)
        cpu.relax_step(dtc, eta)
    for field, ref in (("pos", cpu.pos), ("vel", cpu.vel), ("F", cpu.F), ("alpha", cpu.alpha)):
        err = rel_err(gpu.get(field), ref)
        assert err < 1e-10, (field, err)
    assert np.max(cpu.alpha) > 0, "the bar must reach plastic flow"


def test_config1_membrane2d_run_matches_oracle():
    from oracle import oracle as O
    from oracle.problems import PorousOracle, run_outer_inner as oracle_run
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.stepping import run_outer_inner
    base = resolve({"scenario": "membrane_2d"}).params
    n_outer = 3
    raw = {"scenario": "membrane_2d", "n_outer": n_outer,
           "t_total": n_outer * base["t_total"] / base["n_outer"], "max_inner": 25,
           "min_inner": 25}
    p = resolve(raw).params
    problem, policy = scenarios.build(p, sweep="serial")
    obs, counters = run_outer_inner(problem, policy)
    lat = problem.lattice
    m = O.Membrane(p["density"], p["diffusivity"], p["pressure_coeff"], p["youngs_modulus"],
                   p["poisson_ratio"], p["porosity"], p["fluid_density"], p["initial_saturation"])
    ref = PorousOracle(lat.pos, lat.vol, lat.constrained, lat.contact, m,
                       p["h_factor"] * p["dp"], (1.0, 1.0), p["contact_time"],
                       p["evaporation_rate"], lat.column_id, len(lat.column_x),
                       lat.center_column, lat.deflection_axis)
    rows = oracle_run(ref, policy.dt_outer, n_outer, policy.eta, policy.energy_criterion,
                      cfl=policy.cfl, max_inner=25, min_inner=25)
    np.testing.assert_array_equal(obs.n_inner, [r["n_inner"] for r in rows])
    st = problem.state
    assert np.max(ref.fluid_mass) > 0, "water must enter through the top face"
    assert rel_err(st.fluid_mass, ref.fluid_mass) < 1e-10
    assert rel_err(st.saturation, ref.saturation) < 1e-10
    assert rel_err(st.pos - st.ref_pos, ref.pos - lat.pos) < 1e-8


def _porous_run_vs_oracle(raw, n_outer=3, inner=25):
    """inner: a fixed inner-step count per outer step, or None for the
    reference driver's own protocol (exit on the E_k criterion, capped at
    10 ceil(dt_outer / dt) inner steps, stepping.py:158)."""
    from oracle import oracle as O
    from oracle.problems import PorousOracle, run_outer_inner as oracle_run
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.stepping import run_outer_inner
    base = resolve(raw).params
    raw = dict(raw, n_outer=n_outer, t_total=n_outer * base["t_total"] / base["n_outer"])
    if inner is not None:
        raw.update(max_inner=inner, min_inner=inner)
    p = resolve(raw).params
    problem, policy = scenarios.build(p, sweep="serial")
    obs, counters = run_outer_inner(problem, policy)
    lat = problem.lattice
    m = O.Membrane(p["density"], p["diffusivity"], p["pressure_coeff"], p["youngs_modulus"],
                   p["poisson_ratio"], p["porosity"], p["fluid_density"], p["initial_saturation"])
    ref = PorousOracle(lat.pos, lat.vol, lat.constrained, lat.contact, m,
                       p["h_factor"] * p["dp"], (1.0,) * lat.pos.shape[1], p["contact_time"],
                       p["evaporation_rate"], lat.column_id, len(lat.column_x),
                       lat.center_column, lat.deflection_axis)
    rows = oracle_run(ref, policy.dt_outer, n_outer, policy.eta, policy.energy_criterion,
                      cfl=policy.cfl, max_inner=inner or 0, min_inner=inner or 1)
    np.testing.assert_array_equal(obs.n_inner, [r["n_inner"] for r in rows])
    return problem, ref, lat


@pytest.mark.parametrize("raw,n", [({"scenario": "membrane_2d"}, 8080),
                                   ({"scenario": "membrane_3d", "length": 1.0, "breadth": 0.5}, 6292)])
def test_membrane_configs_reference_protocol(raw, n):
    """BASELINE configs[1] (the whole 2D strip) and the configs[3] plate piece
    through the reference driver's own protocol -- every outer diffusion step
    followed by an inner loop that runs to the kinetic-energy criterion or the
    reference's cap of 10 ceil(dt_outer / dt) steps (90 per outer step on the
    strip), not a fixed short count: the same inner-step counts as the oracle,
    fluid mass and saturation <= 1e-10, displacement <= 1e-8 after four outer
    steps."""
    problem, ref, lat = _porous_run_vs_oracle(raw, n_outer=4, inner=None)
    assert lat.n == n
    st = problem.state
    assert np.max(ref.fluid_mass) > 0
    assert rel_err(st.fluid_mass, ref.fluid_mass) < 1e-10
    assert rel_err(st.saturation, ref.saturation) < 1e-10
    assert rel_err(st.pos - st.ref_pos, ref.pos - lat.pos) < 1e-8


def test_config3_membrane3d_plate_run_matches_oracle():
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    full = resolve({"scenario": "membrane_3d"}).params
    assert abs(lattices.particle_count(full) - 16e6) < 1.5e6       # BASELINE's ~16 M
    problem, ref, lat = _porous_run_vs_oracle({"scenario": "membrane_3d", "length": 1.0,
                                               "breadth": 0.5})
    assert lat.n == 6292
    st = problem.state
    assert np.max(ref.fluid_mass) > 0, "water must enter through the top face"
    assert rel_err(st.fluid_mass, ref.fluid_mass) < 1e-10
    assert rel_err(st.saturation, ref.saturation) < 1e-10
    assert rel_err(st.pos - st.ref_pos, ref.pos - lat.pos) < 1e-8
    # wetting from the top face only: the top layer holds the most water
    z = lat.pos[:, 2]
    assert st.fluid_mass[z == z.max()].mean() > st.fluid_mass[z == z.min()].mean()


def test_config2_slice_serial_trajectory_matches_oracle():
    """A configs[2] slice at full cross-section (0.2 x 2 x 2 at dp 0.02, 100 k
    particles; BASELINE material, right end pulled at the BASELINE rate),
    pre-stretched 0.5 % like the bench so the return map runs its plastic
    branch: 100 inner steps in the reference's damping order (the multi-CTA
    serial kernel at this size) against the oracle, every field <= 1e-10
    (north-star per-step bar)."""
    from oracle.problems import NeckingOracle
    from paper_2309_04010_b200 import device, lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import _necking_materials
    p = resolve({"scenario": "bar_3d", "length": 0.2}).params
    lat = lattices.build_lattice(p)
    assert lat.n == 100_000
    el, hard = _necking_materials(p)
    law, hp = hard.device_params()
    gpu = device.DeviceSolid(lat.pos, lat.vol, el.density0, lat.constrained, lat.side,
                             lat.mid_mask, lat.h_axes, el.shear_modulus, el.bulk_modulus,
                             plastic=True, hardening_law=law, hard=hp, sweep="serial")
    disp = p["stretch_per_end"] / p["n_outer"]           # 1e-5 per outer step
    cpu = NeckingOracle(lat.pos, lat.vol, el.density0, lat.constrained, lat.side < 0,
                        lat.side > 0, lat.mid_mask, el.shear_modulus, el.bulk_modulus, hp,
                        float(lat.h_axes[0]), end_disp_per_outer=disp, ramp_steps=50,
                        hardening_law=law)
    Fm = np.diag([1.005, 1 - 0.3 * 0.005, 1 - 0.3 * 0.005])
    for obj in (gpu, cpu):
        if obj is gpu:
            gpu.set("F", np.broadcast_to(Fm, (lat.n, 3, 3)))
            gpu.set("pos", lat.pos @ Fm.T)
        else:
            cpu.F[:] = Fm
            cpu.pos[:] = lat.pos @ Fm.T
    gpu.set_ramp(disp, 50, 50)
    cpu.advance_slow(1, 0.01, 0.01)
    cfl, eta = p["cfl"], p["eta"]
    for _ in range(100):
        dt = gpu.stable_dt(cfl)
        dtc = cpu.stable_time_step(cfl)
        assert abs(dt - dtc) <= 1e-10 * dtc
        gpu.relax_step(dt, eta)
        cpu.relax_step(dtc, eta)
    for field, ref in (("pos", cpu.pos), ("vel", cpu.vel), ("F", cpu.F), ("alpha", cpu.alpha)):
        err = rel_err(gpu.get(field), ref)
        assert err < 1e-10, (field, err)
    assert np.mean(cpu.alpha > 0) > 0.5, "the slice must be in plastic flow"
