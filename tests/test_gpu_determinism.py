"""GPU: run-level determinism, the counterpart of the reference's
byte-identical-CSV test (test_acceptance.py:409-435).  The same configs are
run twice through the drop-in driver; every observable series and the final
state must be bitwise equal.  Covered for the reference order (serial) and
both parallel orders: the tiled sweep's persistent dataflow launch claims
block tasks from a global counter in whatever order CTAs arrive, and the
schedule makes that order irrelevant to the result; the reductions are
fixed-order block trees."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

NECK = {"scenario": "necking_2d", "length": 8e-3, "width": 2e-3, "dp": 0.5e-3,
        "stretch_per_end": 1e-5, "n_outer": 5, "ramp_steps": 5, "max_inner": 60,
        "energy_ref": 1e-3}
FSI = {"scenario": "fsi_2d", "length": 2e-3, "t_total": 2.4, "n_outer": 3,
       "contact_time": 0.8, "max_inner": 40}
BLOCK = {"scenario": "block_3d", "length": 0.4, "width": 0.2, "breadth": 0.2,
         "stretch_per_end": 1e-3, "n_outer": 3, "max_inner": 80}


def _run(raw, sweep):
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.stepping import run_outer_inner
    problem, policy = scenarios.build(resolve(raw).params, sweep=sweep)
    obs, counters = run_outer_inner(problem, policy)
    series = {k: getattr(obs, k) for k in ("time", "reaction_force", "neck_disp", "amplitude",
                                           "ek_ratio", "n_inner", "ns_cum", "nd_cum")}
    series.update({f"x_{k}": np.asarray(v) for k, v in obs.extras.items()})
    fields = ("pos", "vel", "F") if raw["scenario"] != "fsi_2d" else \
        ("pos", "vel_solid", "F", "fluid_mass", "saturation")
    state = {f: problem.dev.get(f) for f in fields}
    return series, state


@pytest.mark.parametrize("raw", [NECK, FSI, BLOCK], ids=["necking_2d", "fsi_2d", "block_3d"])
@pytest.mark.parametrize("sweep", ["serial", "tiled", "coloured"])
def test_repeated_runs_are_bitwise_identical(raw, sweep):
    if raw is BLOCK and sweep == "serial":
        pytest.skip("covered by the 2D runs; the 3D serial order is the slow parity mode")
    a, sa = _run(raw, sweep)
    b, sb = _run(raw, sweep)
    assert a.keys() == b.keys()
    for k in a:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)
    for k in sa:
        assert sa[k].tobytes() == sb[k].tobytes(), k
    assert np.sum(a["n_inner"]) > 0
