"""GPU: the parallel damping orders against the reference's serial order.

The coloured (midpoint-cell tasks) and tiled (shared-memory blocks)
sweeps apply the same closed-form pair updates as the reference in a
different deterministic order, so:
  * damping alone conserves total momentum and never raises kinetic
    energy (checked on a free body where stress forces are negligible);
  * whole relaxations reach the same equilibrium as the serial order:
    final displacement and stress fields within 1e-5 relative L2
    (north-star bound), on elastic and elastoplastic bars.
"""

import numpy as np
import pytest

from conftest import jittered_lattice

pytestmark = pytest.mark.gpu

SWEEPS = ["serial", "coloured", "tiled"]


@pytest.mark.parametrize("sweep", SWEEPS)
@pytest.mark.parametrize("dim", [2, 3])
def test_damping_conserves_momentum_and_dissipates(sweep, dim):
    from paper_2309_04010_b200.device import DeviceSolid
    pos, vol = jittered_lattice(14 if dim == 2 else 8, dim, dp=0.01, jitter=0.05, seed=5)
    n = len(vol)
    rng = np.random.default_rng(7)
    s = DeviceSolid(pos, vol, 2.0, np.zeros(n, bool), np.zeros(n, np.int8), None,
                    [1.35 * 0.01] * dim, 1e-12, 1e-12, plastic=False, sweep=sweep)
    mass = 2.0 * vol
    vel = rng.normal(size=(n, dim))
    s.set("vel", vel)
    p0 = mass @ vel
    e0 = 0.5 * np.sum(mass[:, None] * vel * vel)
    for _ in range(20):
        s.relax_step(1e-9, 1e7)
        v = s.get("vel")
        e = 0.5 * np.sum(mass[:, None] * v * v)
        assert e <= e0 * (1 + 1e-13)
        e0 = e
    p1 = mass @ s.get("vel")
    scale = np.sum(mass * np.linalg.norm(vel, axis=1))
    assert np.max(np.abs(p1 - p0)) <= 1e-12 * scale
    assert e0 < 0.5 * 0.5 * np.sum(mass[:, None] * vel * vel)   # it did damp


@pytest.mark.parametrize("dim", [2, 3])
def test_tiled_pipeline_matches_serial_pipeline_without_damping(dim):
    """With eta = 0 the sweep is the identity, so a solid built for the tiled
    sweep (block schedule, dataflow launch) must track one built for the
    serial sweep step by step."""
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.device import DeviceSolid
    from paper_2309_04010_b200.scenarios import _necking_materials
    raw = {"scenario": "block_3d", "length": 0.3, "width": 0.16, "breadth": 0.16, "dp": 0.02} \
        if dim == 3 else {"scenario": "bar_2d", "length": 2.0, "width": 0.6, "dp": 0.05}
    p = resolve(raw).params
    lat = lattices.build_lattice(p)
    el, hard = _necking_materials(p)
    law, hp = hard.device_params()
    runs = {}
    for sweep in ("serial", "tiled"):
        s = DeviceSolid(lat.pos, lat.vol, el.density0, lat.constrained, lat.side, lat.mid_mask,
                        lat.h_axes, el.shear_modulus, el.bulk_modulus, plastic=True,
                        hardening_law=law, hard=hp, sweep=sweep)
        s.set_ramp(0.01 * p["length"], 20, 20)
        hist = []
        for _ in range(40):
            dt = s.stable_dt(0.2)
            s.relax_step(dt, 0.0)
            hist.append(dt)
        runs[sweep] = (hist, s.get("pos") - lat.pos, s.get("vel"), s.get("F"), s.get("alpha"))
    a, b = runs["serial"], runs["tiled"]
    np.testing.assert_allclose(a[0], b[0], rtol=1e-10)
    for x, y in zip(a[1:], b[1:]):
        scale = max(np.max(np.abs(x)), 1e-300)
        assert np.max(np.abs(x - y)) <= 1e-10 * scale
    assert np.max(a[4]) > 0, "case must yield"


@pytest.mark.parametrize("dim", [2, 3])
def test_dataflow_sweep_is_bit_identical_to_colour_launches(dim, monkeypatch):
    """The persistent dataflow sweep (one launch, blocks start as their
    overlapping neighbours of earlier phases finish) applies the same updates
    in the same order on every particle as the per-colour launches."""
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.device import DeviceSolid
    from paper_2309_04010_b200.scenarios import _necking_materials
    raw = {"scenario": "block_3d", "length": 0.6, "width": 0.3, "breadth": 0.3, "dp": 0.02} \
        if dim == 3 else {"scenario": "bar_2d", "length": 4.0, "width": 1.0, "dp": 0.02}
    p = resolve(raw).params
    lat = lattices.build_lattice(p)
    el, hard = _necking_materials(p)
    law, hp = hard.device_params()
    runs = {}
    for flow in ("1", "0"):
        monkeypatch.setenv("MTSPH_SWEEP_FLOW", flow)
        s = DeviceSolid(lat.pos, lat.vol, el.density0, lat.constrained, lat.side, lat.mid_mask,
                        lat.h_axes, el.shear_modulus, el.bulk_modulus, plastic=True,
                        hardening_law=law, hard=hp, sweep="tiled")
        s.set_ramp(0.01 * p["length"], 10, 10)
        for _ in range(30):
            s.relax_step(s.stable_dt(0.2), p["eta"])
        runs[flow] = [s.get(f) for f in ("pos", "vel", "F", "alpha")]
    for x, y in zip(runs["1"], runs["0"]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("dim", [2, 3])
def test_serial_sweep_shared_memory_kernel_is_bit_identical(dim, monkeypatch):
    """The reference-order sweep of small problems runs from shared memory
    (velocities and level table staged, pair entries prefetched); it applies
    the same operations in the same order as the global-memory kernel."""
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.device import DeviceSolid
    from paper_2309_04010_b200.scenarios import _necking_materials
    raw = {"scenario": "block_3d", "length": 0.2, "width": 0.08, "breadth": 0.08, "dp": 0.01} \
        if dim == 3 else {"scenario": "bar_2d", "length": 2.0, "width": 0.4, "dp": 0.025}
    p = resolve(raw).params
    lat = lattices.build_lattice(p)
    el, hard = _necking_materials(p)
    law, hp = hard.device_params()
    runs = {}
    for smem in ("1", "0"):
        monkeypatch.setenv("MTSPH_SERIAL_SMEM", smem)
        s = DeviceSolid(lat.pos, lat.vol, el.density0, lat.constrained, lat.side, lat.mid_mask,
                        lat.h_axes, el.shear_modulus, el.bulk_modulus, plastic=True,
                        hardening_law=law, hard=hp, sweep="serial")
        s.set_ramp(0.01 * p["length"], 10, 10)
        for _ in range(30):
            s.relax_step(s.stable_dt(0.2), p["eta"])
        r = s.relax(eta=p["eta"], cfl=p["cfl"], criterion=-1.0, dt_outer=1.0, max_inner=20,
                    min_inner=20)
        assert r.n_inner == 20
        runs[smem] = [s.get(f) for f in ("pos", "vel", "F", "alpha")]
    assert np.max(np.abs(runs["1"][1])) > 0
    for x, y in zip(runs["1"], runs["0"]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("case", ["block3d", "bar2d", "fsi2d"])
def test_serial_sweep_multi_cta_kernel_is_bit_identical(case, monkeypatch):
    """The multi-CTA reference-order kernel (levels spread over the grid, a
    grid barrier between levels) applies the same operations in the same
    order as the one-CTA global kernel: bitwise equal state after a loaded
    run, for the solid in 3D and 2D and for the membrane (simultaneous
    group solves)."""
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import build
    from paper_2309_04010_b200.stepping import run_outer_inner
    raw = {"block3d": {"scenario": "block_3d", "length": 0.4, "width": 0.2, "breadth": 0.2,
                       "dp": 0.01, "stretch_per_end": 4e-3, "n_outer": 2, "max_inner": 40},
           "bar2d": {"scenario": "bar_2d", "length": 4.0, "width": 0.8, "dp": 0.025,
                     "stretch_per_end": 0.02, "n_outer": 2, "max_inner": 60},
           "fsi2d": {"scenario": "fsi_2d", "length": 2e-3, "t_total": 2.4, "n_outer": 3,
                     "max_inner": 40}}[case]
    p = resolve(raw).params
    monkeypatch.setenv("MTSPH_SERIAL_SMEM", "0")
    runs = {}
    for grid in ("1", "0"):
        monkeypatch.setenv("MTSPH_SERIAL_GRID", grid)
        problem, policy = build(p, sweep="serial")
        obs, _ = run_outer_inner(problem, policy)
        vel = "vel_solid" if case == "fsi2d" else "vel"
        runs[grid] = (obs.n_inner, [problem.dev.get(f) for f in ("pos", vel, "F")])
    np.testing.assert_array_equal(runs["1"][0], runs["0"][0])
    assert np.max(np.abs(runs["1"][1][1])) > 0
    for x, y in zip(runs["1"][1], runs["0"][1]):
        np.testing.assert_array_equal(x, y)


def test_serial_sweep_shared_memory_kernel_is_bit_identical_porous(monkeypatch):
    """Same for the membrane (anisotropic kernel, simultaneous group solves
    included where the reference groups pairs)."""
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import build
    from paper_2309_04010_b200.stepping import run_outer_inner
    p = resolve({"scenario": "fsi_2d", "length": 2e-3, "t_total": 2.4, "n_outer": 3,
                 "max_inner": 40}).params
    runs = {}
    for smem in ("1", "0"):
        monkeypatch.setenv("MTSPH_SERIAL_SMEM", smem)
        problem, policy = build(p, sweep="serial")
        obs, _ = run_outer_inner(problem, policy)
        runs[smem] = (obs.n_inner, [problem.dev.get(f) for f in ("pos", "vel_solid", "fluid_mass")])
    np.testing.assert_array_equal(runs["1"][0], runs["0"][0])
    assert np.max(np.abs(runs["1"][1][1])) > 0
    for x, y in zip(runs["1"][1], runs["0"][1]):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("flow", ["1", "0"])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("shape", ["tiny", "thin"])
def test_tiled_sweep_degenerate_problems(shape, dim, flow, monkeypatch):
    """Smallest valid bodies (2^d particles: one block, one cell) and a thin
    bar one to two particles wide (many blocks, most colours empty) through
    both tiled launch modes: no failure, damping still conserves momentum
    and never adds energy.  (A lone or collinear particle set is rejected
    like in the reference: singular kernel moment matrix.)"""
    from paper_2309_04010_b200.device import DeviceSolid
    monkeypatch.setenv("MTSPH_SWEEP_FLOW", flow)
    rng = np.random.default_rng(dim)
    dp = 0.01
    counts = [2] * dim if shape == "tiny" else [60] + [2] * (dim - 1)
    grids = np.meshgrid(*[np.arange(c) * dp for c in counts], indexing="ij")
    pos = np.stack(grids, -1).reshape(-1, dim) + rng.uniform(-1e-4, 1e-4, (int(np.prod(counts)), dim))
    n = len(pos)
    vol = np.full(n, dp ** dim)
    s = DeviceSolid(pos, vol, 1.0, np.zeros(n, bool), np.zeros(n, np.int8), None,
                    [1.3 * dp] * dim, 1e-12, 1e-12, plastic=False, sweep="tiled")
    vel = rng.normal(size=(n, dim))
    s.set("vel", vel)
    mass = vol * 1.0
    e0 = 0.5 * np.sum(mass[:, None] * vel * vel)
    for _ in range(5):
        s.relax_step(1e-9, 1e6)
    v = s.get("vel")
    assert np.all(np.isfinite(v))
    assert np.max(np.abs(mass @ v - mass @ vel)) <= 1e-12 * np.sum(mass * np.linalg.norm(vel, axis=1))
    assert 0.5 * np.sum(mass[:, None] * v * v) <= e0 * (1 + 1e-13)


def _relaxed(raw, sweep):
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = scenarios.build(resolve(raw).params, sweep=sweep)
    obs, counters = run_outer_inner(problem, policy)
    st = problem.state
    return st.pos - st.ref_pos, problem._accel, problem.dev.get("F"), counters


def test_parallel_sweeps_reach_the_serial_equilibrium():
    """Elastic equilibria are unique: every damping order relaxes a loaded
    elastic bar to the serial (reference) order's equilibrium within the
    north star's 1e-5."""
    raw = {"scenario": "necking_2d", "length": 8e-3, "width": 2e-3, "dp": 0.5e-3,
           "plasticity": False, "stretch_per_end": 4e-6, "n_outer": 3, "ramp_steps": 10,
           "energy_ref": 1.0, "energy_pct": 1e-17, "max_inner": 40000}
    u_ref, _, f_ref, c_ref = _relaxed(raw, "serial")
    assert not c_ref.cap_hits
    for sweep in ("coloured", "tiled"):
        u, _, f, c = _relaxed(raw, sweep)
        assert not c.cap_hits
        du = np.linalg.norm(u - u_ref) / np.linalg.norm(u_ref)
        df = np.linalg.norm(f - f_ref) / np.linalg.norm(f_ref - np.eye(u.shape[1]))
        assert du < 1e-5 and df < 1e-5, (sweep, du, df)


def _baseline_loading(raw, sweep, pre, pre_ramp, pre_max, n_outer):
    """BASELINE loading through the drop-in driver protocol: a slow ramp to
    `pre` x the yield end displacement (sigma0 / E x length; elastic, so the
    state does not depend on how it was reached), then n_outer outer steps of
    the BASELINE pull (1e-3 length units per unit time, outer dt 0.01, the
    ramp over 50 inner steps, inner loop to E_k <= 1e-8 or the reference's
    cap), then relaxation to E_k <= 1e-8."""
    from oracle import oracle as O
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    p = resolve(raw).params
    prob, pol = scenarios.build(p, sweep=sweep)
    dev = prob.dev
    e_mod = 9 * p["bulk_modulus"] * p["shear_modulus"] / (3 * p["bulk_modulus"] + p["shear_modulus"])
    dev.set_ramp(pre * p["initial_flow_stress"] / e_mod * p["length"], pre_ramp, pre_ramp)
    dev.relax(pol.eta, pol.cfl, pol.energy_criterion, pol.dt_outer, max_inner=pre_max, min_inner=1)
    for step in range(1, n_outer + 1):
        prob.advance_slow(step, pol.dt_outer, step * pol.dt_outer)
        prob.relax_inner(pol)
    r = dev.relax(pol.eta, pol.cfl, pol.energy_criterion, pol.dt_outer, max_inner=400000, min_inner=1)
    assert not r.cap_hit and r.ek <= pol.energy_criterion
    F, cp, alpha = dev.get("F"), dev.get("cp_inv"), dev.get("alpha")
    law, hp = scenarios._necking_materials(p)[1].device_params()
    matp = O.material_vector(p["shear_modulus"], p["bulk_modulus"], *hp, law=law)
    tau = O.return_map(F, cp, alpha, matp)[0]      # stress of the relaxed state
    return {"u": dev.get("pos") - prob.lattice.pos, "tau": tau, "F": F - np.eye(F.shape[1]),
            "alpha": alpha}


@pytest.mark.parametrize("case", ["config0_bar2d", "config2_material_block3d"])
def test_tiled_order_meets_the_equilibrium_bar_under_baseline_loading(case):
    """The benchmarked (tiled) damping order against the reference's serial
    order through first yield under the BASELINE loading: displacement,
    Kirchhoff stress and F of the relaxed states <= 1e-5 relative L2 (north
    star).  configs[0] itself (the 20 x 2 bar, 4000 particles), and a
    0.4^3 block of configs[2]'s material, dp and loading (8000 particles).
    Plastic flow covers most of the body by the end (asserted)."""
    raw, pre, pre_ramp, pre_max, n_outer, plastic = {
        "config0_bar2d": ({"scenario": "bar_2d"}, 0.98, 3000, 6000, 200, 0.3),
        "config2_material_block3d": ({"scenario": "bar_3d", "length": 0.4, "width": 0.4,
                                      "breadth": 0.4}, 0.95, 4000, 8000, 40, 0.5),
    }[case]
    ref = _baseline_loading(raw, "serial", pre, pre_ramp, pre_max, n_outer)
    got = _baseline_loading(raw, "tiled", pre, pre_ramp, pre_max, n_outer)
    assert np.mean(ref["alpha"] > 0) > plastic, np.mean(ref["alpha"] > 0)
    diffs = {k: float(np.linalg.norm(got[k] - ref[k]) / np.linalg.norm(ref[k])) for k in ("u", "tau", "F")}
    print(case, "tiled vs serial relative L2:", diffs,
          "plastic fraction", float(np.mean(ref["alpha"] > 0)))
    for k, d in diffs.items():
        assert d <= 1e-5, (k, d)


@pytest.mark.parametrize("bits", [64, 32])
def test_full_size_bench_workload_damping_invariants(bits):
    """The benchmark's own 10 M-particle bar (BASELINE configs[2] geometry):
    size-independent properties of the tiled damping sweep at full size --
    with the elastic forces switched off (moduli 1e-30) the inner step is
    kick/drift + damping, so total momentum is conserved to rounding and the
    kinetic energy never increases, in fp64 and in the fp32 variant."""
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.device import DeviceSolid
    p = resolve({"scenario": "bar_3d", "damping_sweep": "tiled"}).params
    lat = lattices.build_lattice(p)
    n = lat.n
    assert n == 10_000_000
    free = np.zeros(n, bool)
    s = DeviceSolid(lat.pos, lat.vol, 1.0, free, np.zeros(n, np.int8), None, lat.h_axes,
                    1e-30, 1e-30, plastic=False, sweep="tiled")
    rng = np.random.default_rng(11)
    vel = rng.normal(size=(n, 3))
    s.set("vel", vel)
    s.set_precision(bits)
    mass = lat.vol * 1.0
    v0 = s.get("vel")
    p0 = mass @ v0
    e0 = 0.5 * float(np.sum(mass[:, None] * v0 * v0))
    first = e0
    for _ in range(3):
        s.relax_step(1e-9, 1e7)
        v = s.get("vel")
        e = 0.5 * float(np.sum(mass[:, None] * v * v))
        assert e <= e0 * (1 + (1e-12 if bits == 64 else 1e-6))
        e0 = e
    scale = float(np.sum(mass * np.linalg.norm(vel, axis=1)))
    tol = 1e-12 if bits == 64 else 1e-6
    assert np.max(np.abs(mass @ s.get("vel") - p0)) <= tol * scale
    assert e0 < 0.5 * first
