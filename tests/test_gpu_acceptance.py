"""GPU: the reference's physical acceptance criteria
(/root/reference/pkg/tests/test_acceptance.py), restated against this
package's drop-in driver (scenarios.build + stepping.run_outer_inner, the
inner loops on the device), plus parity with the reference's own runs of
those configurations (tests/golden/acceptance_heads.npz, made by
tests/golden/make_golden.py from the real reference):

  * parity: the first 12 outer steps of the desk necking bar (through
    first mid-span yield) and the whole 125-step paper-scale FSI membrane
    run, reference damping order -- inner-step counts exact, every
    observable series (the deflection profiles included) and the final
    state to 1e-9;
  * 2D necking bar at desk resolution (dp = PH/25, 1000 outer steps;
    test_acceptance.py:243-305), run with the B200 tiled damping order:
    the neck forms at mid-span, the force curve rises linearly, peaks once
    and falls, first mid-span yield within 15 % of sigma0 * A, every inner
    loop ends under the 0.5 % criterion, and the multi-rate loop needs
    >= 100x fewer inner steps than a single-rate run;
  * 2D FSI membrane at paper scale (125 outer steps;
    test_acceptance.py:320-405): saturation within [0, porosity], the
    deflection profile mirror-symmetric to 1e-6, the amplitude rising
    through the contact window and the profile not narrowing afterwards, the
    post-contact fluid mass drift <= 1 %, the wetted region only losing
    water after contact.
Three reference criteria are not asserted as written, because the
reference's own run does not meet them at these settings (fixture
af2_*): the amplitude at 9.6 s is 1.063x the first sample (the criterion
asks for 5x), and the half-maximum width of the profile is 57 columns both
at 9.6 s and at 100 s (the criterion asks for a strict increase) -- here
both are asserted equal to the reference's values, which the run matches to
1e-14; the drift comparison against a 16x finer run (500 outer steps of
~20k particles, beyond the CPU reference in this container) is not made.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DESK_DP = 12.826e-3 / 25     # the reference's desk resolution (PH / 25)


@pytest.fixture(scope="module")
def desk_necking():
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import build
    from paper_2309_04010_b200.stepping import run_outer_inner
    params = resolve({"scenario": "necking_2d", "dp": DESK_DP, "n_outer": 1000}).params
    problem, policy = build(params, sweep="tiled")
    obs, counters = run_outer_inner(problem, policy)
    return {"obs": obs, "counters": counters, "problem": problem, "params": params}


def test_necking_localizes_at_midspan(desk_necking):
    st = desk_necking["problem"].state
    ref_x, pos = st.ref_pos[:, 0], st.pos
    cols = np.unique(np.round(ref_x, 9))
    widths, xs = [], []
    for c in cols:
        sel = np.isclose(ref_x, c)
        widths.append(np.ptp(pos[sel, 1]))
        xs.append(np.mean(pos[sel, 0]))
    assert abs(xs[int(np.argmin(widths))]) <= 2.0 * DESK_DP


def test_necking_force_curve_shape(desk_necking):
    obs = desk_necking["obs"]
    force = obs.reaction_force
    peak = float(np.max(force))
    smooth = np.convolve(force, np.ones(9) / 9.0, mode="valid")
    ipk = int(np.argmax(smooth))
    assert 0 < ipk < len(smooth) - 1
    assert np.all(np.diff(smooth[:ipk]) > -1e-3 * peak)
    assert np.all(np.diff(smooth[ipk:]) < 1e-3 * peak)
    assert smooth[-1] < 0.95 * peak
    t = obs.time
    fit = np.polyfit(t[1:8], force[1:8], 1)
    assert np.max(np.abs(np.polyval(fit, t[1:8]) - force[1:8])) < 0.02 * force[7]


def test_necking_initial_yield_force(desk_necking):
    obs = desk_necking["obs"]
    iy = int(np.argmax(obs.extras["mid_alpha_min"] > 0.0))
    assert iy > 0
    sigma0_a = 450e6 * 12.826e-3          # plane strain, unit thickness
    assert abs(obs.reaction_force[iy] - sigma0_a) <= 0.15 * sigma0_a


def test_necking_energy_criterion_and_iteration_reduction(desk_necking):
    obs, counters = desk_necking["obs"], desk_necking["counters"]
    assert not counters.cap_hits
    assert np.all(obs.ek_ratio <= 0.005 * (1.0 + 1e-12))
    ratio = counters.single_rate_baseline(desk_necking["params"]["t_total"]) / counters.n_inner
    print(f"inner steps {counters.n_inner}, single-rate baseline / inner = {ratio:.0f}")
    assert ratio >= 100.0


@pytest.fixture(scope="module")
def fsi_2d_run():
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import build
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = build(resolve({"scenario": "fsi_2d"}).params)
    profiles = []
    obs, counters = run_outer_inner(problem, policy,
                                    observers=[lambda s, t, smp: profiles.append(smp["profile"])])
    return {"obs": obs, "counters": counters, "problem": problem,
            "profiles": np.array(profiles)}


def test_fsi_outer_steps_and_saturation_bounds(fsi_2d_run):
    assert fsi_2d_run["counters"].n_outer == 125
    assert np.all(fsi_2d_run["obs"].extras["max_saturation"] <= 0.4 * (1 + 1e-12))
    sat = fsi_2d_run["problem"].state.saturation
    assert np.all(sat >= 0.0) and np.all(sat <= 0.4 * (1 + 1e-12))


def test_fsi_deflection_symmetry(fsi_2d_run):
    prof = fsi_2d_run["profiles"]
    assert np.max(np.abs(prof - prof[:, ::-1])) <= 1e-6 * np.max(np.abs(prof))


def test_fsi_amplitude_pattern(fsi_2d_run, gold_accept):
    obs = fsi_2d_run["obs"]
    prof = np.abs(fsi_2d_run["profiles"])
    i10 = int(np.searchsorted(obs.time, 10.0))
    amp = np.abs(obs.amplitude)
    ref = np.abs(gold_accept["af2_amplitude"])
    assert amp[i10 - 1] / amp[0] == pytest.approx(ref[i10 - 1] / ref[0], rel=1e-9)
    assert amp[i10 - 1] > amp[0]
    assert np.all(np.diff(amp[:i10]) > -1e-9 * amp[i10 - 1])

    def half_width(p):
        return np.count_nonzero(p > 0.5 * p.max())

    ref_prof = np.abs(gold_accept["af2_profile"])
    assert (half_width(prof[-1]), half_width(prof[i10 - 1])) == \
        (half_width(ref_prof[-1]), half_width(ref_prof[i10 - 1]))
    assert half_width(prof[-1]) >= half_width(prof[i10 - 1])


def test_fsi_fluid_mass_drift(fsi_2d_run):
    obs = fsi_2d_run["obs"]
    mass = obs.extras["fluid_mass_total"]
    first = int(np.searchsorted(obs.time, 10.0 * (1 + 1e-9), "right"))
    drift = abs(mass[-1] - mass[first]) / mass[first]
    print(f"post-contact fluid mass drift {drift:.2e}")
    assert drift <= 0.01
    i10 = int(np.searchsorted(obs.time, 10.0))
    region = obs.extras["contact_mass_total"]
    assert np.all(np.diff(region[i10:]) <= 1e-12 * region[i10])


# ---------------------------------------------------------------- parity

@pytest.fixture(scope="module")
def gold_accept():
    from conftest import golden
    return golden("acceptance_heads.npz")


SERIES = {"an2_": ("reaction_force", "neck_disp", "max_alpha", "mid_alpha_min", "ek_ratio"),
          "af2_": ("amplitude", "fluid_mass_total", "contact_mass_total", "max_saturation",
                   "ek_ratio", "profile")}


def _check_run(prefix, obs, problem, gold):
    from conftest import rel_err
    np.testing.assert_array_equal(obs.n_inner, gold[prefix + "n_inner"])
    for key in SERIES[prefix]:
        got = getattr(obs, key) if hasattr(obs, key) else obs.extras[key]
        want = gold[prefix + key]
        scale = max(float(np.max(np.abs(want))), 1e-300)
        err = float(np.max(np.abs(got - want))) / scale
        print(prefix + key, f"{err:.2e}")
        assert err < 1e-9, (key, err)
    st = problem.state
    assert rel_err(st.pos - st.ref_pos, gold[prefix + "pos"] - st.ref_pos) < 1e-9
    if prefix == "an2_":
        assert rel_err(problem.plastic.alpha, gold["an2_alpha"]) < 1e-9
    else:
        assert rel_err(st.fluid_mass, gold["af2_fluid_mass"]) < 1e-9
        assert rel_err(st.saturation, gold["af2_saturation"]) < 1e-9


def test_desk_necking_head_matches_reference_run(gold_accept):
    """First 12 outer steps (through first mid-span yield), reference order."""
    import dataclasses
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import build
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = build(resolve({"scenario": "necking_2d", "dp": DESK_DP,
                                     "n_outer": 1000}).params)
    n_outer = len(gold_accept["an2_n_inner"])
    obs, _ = run_outer_inner(problem, dataclasses.replace(policy, n_outer=n_outer))
    assert np.max(gold_accept["an2_mid_alpha_min"]) > 0, "the fixture covers mid-span yield"
    _check_run("an2_", obs, problem, gold_accept)


def test_fsi_paper_run_matches_reference_run(fsi_2d_run, gold_accept):
    """The whole 125-step paper-scale membrane run against the reference's."""
    _check_run("af2_", fsi_2d_run["obs"], fsi_2d_run["problem"], gold_accept)
