"""GPU: conservation properties of the device solid step, restated from the
reference's own tests (files under /root/reference/pkg/tests):

  * test_solids.py:225 (free-body drift): a free elastic body stepped
    without damping keeps its total momentum to round-off over 1000 inner
    steps -- the acceleration (T_a + T_b) . gradW_ab is antisymmetric pair
    by pair, so its mass-weighted sum vanishes;
  * test_stepping.py:52 / :96 (pair and total momentum): with damping
    on, the implicit pairwise exchange conserves momentum as well, in
    either sweep order.
Both in 2D and 3D on jittered lattices, fp64.
"""

import numpy as np
import pytest

from conftest import jittered_lattice

pytestmark = pytest.mark.gpu

MU, K, RHO = 80.1938e9, 164.21e9, 7850.0    # the reference's steel


def _free_body(dim, sweep, seed):
    from paper_2309_04010_b200.device import DeviceSolid
    n_side = 8 if dim == 2 else 6
    dp = 1e-3
    pos, vol = jittered_lattice(n_side, dim, dp=dp, jitter=0.05, seed=seed)
    n = len(vol)
    s = DeviceSolid(pos, vol, RHO, np.zeros(n, bool), np.zeros(n, np.int8), None,
                    [1.3 * dp] * dim, MU, K, plastic=False, sweep=sweep)
    vel = 1e-3 * np.random.default_rng(seed).normal(size=(n, dim))
    s.set("vel", vel)
    return s, RHO * vol, vel


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("sweep,eta", [("serial", 0.0), ("serial", 1e4), ("tiled", 1e4)])
def test_free_body_momentum_drift(dim, sweep, eta):
    s, mass, vel = _free_body(dim, sweep, seed=23)
    p0 = mass @ vel
    for _ in range(1000):
        s.relax_step(s.stable_dt(0.6), eta)
    v1 = s.get("vel")
    assert np.max(np.abs(v1 - vel)) > 0, "the body must deform"
    p1 = mass @ v1
    scale = np.sum(mass * np.linalg.norm(v1, axis=1))
    assert np.max(np.abs(p1 - p0)) <= 1e-11 * scale
    # the step's acceleration field itself sums to zero momentum
    a = s.get("accel")
    assert np.max(np.abs(mass @ a)) <= 1e-11 * np.sum(mass * np.linalg.norm(a, axis=1))
