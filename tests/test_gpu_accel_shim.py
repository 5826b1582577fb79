"""GPU: the committed ``_accel`` drop-in (paper_2309_04010_b200/accel.py).

1. Every function, called exactly like the reference calls its numba twin,
   on the reference's own arrays (golden neighbourhoods) reproduces the
   reference's outputs.
2. The reference's NeckingProblem.relax_step (scenarios.py:113-141), with
   every kernel call of its call chain -- deformation_rate
   (solids.py:118 -> velocity_gradient_gather), stress_divergence_acceleration
   (solids.py:170 -> pair_tensor_divergence) and apply_damping_sweep
   (stepping.py:101 -> damping_sweep) -- routed through the shim, reproduces
   the reference's own 100-step plastic necking trajectories (golden
   fixture) to 1e-10 at steps 1, 10, 50, 100 in 2D and 3D.  The return map
   is the oracle's restatement of plasticity.py:118 (pinned separately); it
   is not an _accel kernel.
"""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


def _nb(gold_nbh, nb):
    return {k[len(nb):]: gold_nbh[k] for k in gold_nbh.files if k.startswith(nb)}


@pytest.mark.parametrize("op,nb", [("op2d_", "nbh2d_"), ("op3d_", "nbh3d_")])
def test_shim_gathers_and_sweep_match_reference(gold_nbh, gold_ops, op, nb):
    from paper_2309_04010_b200 import accel
    g = _nb(gold_nbh, nb)
    n, d = g["pos"].shape
    raw = np.empty((n, d, d))
    accel.velocity_gradient_gather(gold_ops[op + "vel"], g["indptr"], g["idx"], g["grad0"],
                                   g["vol"], raw)
    assert rel_err(raw @ g["corr"], gold_ops[op + "rate"]) < 1e-13
    out = np.empty((n, d))
    accel.pair_tensor_divergence(np.ascontiguousarray(gold_ops[op + "pk1"] @ g["corr"]),
                                 g["indptr"], g["idx"], g["grad0"], g["vol"], out)
    assert rel_err(out / 7850.0, gold_ops[op + "acc"]) < 1e-13
    # in-place sweep on a non-contiguous view (numba writes through views)
    inv = np.where(gold_ops[op + "movable"], 1.0 / gold_ops[op + "mass"], 0.0)
    big = np.zeros((n, d + 1))
    vel = big[:, :d]
    vel[...] = gold_ops[op + "damp_vin"]
    accel.damping_sweep(vel, g["pair_i"], g["pair_j"], g["pair_damp"], inv[g["pair_i"]],
                        inv[g["pair_j"]], g["pair_group"], 1e3, 1e-3)
    assert rel_err(vel, gold_ops[op + "damp_vout"]) < 1e-14
    assert np.all(big[:, d] == 0.0)


@pytest.mark.parametrize("p", ["p2d_", "p3d_"])
def test_shim_porous_kernels_match_reference(gold_porous, p):
    from oracle import oracle as O
    from paper_2309_04010_b200 import accel
    gp = gold_porous
    pos, vol = gp[p + "pos"], gp[p + "vol"]
    n, d = pos.shape
    nbh = O.build_nbh(pos, vol, 1.35e-5)
    F = gp[p + "F"]
    m = O.Membrane(*gp["model"])
    volc = vol * np.linalg.det(F)
    amap = np.linalg.inv(F) @ np.swapaxes(nbh.corr, -1, -2)
    rho_l = gp[p + "mass_in"] / volc
    q = np.empty((n, d))
    accel.scalar_difference_flux(rho_l / m.fluid_density0, m.diffusivity * rho_l, amap,
                                 nbh.indptr, nbh.idx, volc, nbh.grad0, q)
    assert rel_err(q, gp[p + "q"]) < 1e-13
    rate = np.empty(n)
    accel.conservative_mass_rate(gp[p + "flux_in"], amap, nbh.pair_i, nbh.pair_j,
                                 nbh.pair_grad, volc, rate)
    mass = np.clip(gp[p + "mass_in"] + 50.0 * rate, 0.0, m.porosity * m.fluid_density0 * volc)
    assert rel_err(mass, gp[p + "mass_out"]) < 1e-13
    tbuf, jout, srate = np.empty((n, d, d)), np.empty(n), np.empty((n, d))
    accel.porous_stress_rhs(F, gp[p + "pressure"], nbh.corr, nbh.indptr, nbh.idx, nbh.grad0,
                            vol, m.mu, m.lam, tbuf, jout, srate)
    assert rel_err(tbuf, gp[p + "tbuf"]) < 1e-13
    assert rel_err(srate, gp[p + "stress_rate"]) < 1e-13
    frate = np.zeros((n, d))
    accel.pair_tensor_divergence_mapped(gp[p + "vel_fluid"][:, :, None] * gp[p + "flux_in"][:, None, :],
                                        -amap, nbh.indptr, nbh.idx, nbh.grad0, volc, frate)
    assert rel_err(frate, gp[p + "flux_rate"]) < 1e-13


class _ReferenceStep:
    """NeckingProblem.relax_step (reference scenarios.py:113-141) with its
    _accel calls bound to the shim; numpy glue as in the reference."""

    def __init__(self, pos, vol, constrained, dp, accel):
        from oracle import oracle as O
        self.O, self.accel = O, accel
        n, d = pos.shape
        self.nbh = O.build_nbh(pos, vol, 1.35 * dp)
        self.pos = pos.copy()
        self.vel = np.zeros((n, d))
        self.F = np.broadcast_to(np.eye(d), (n, d, d)).copy()
        self.cp = self.F.copy()
        self.alpha = np.zeros(n)
        self.acc = np.zeros((n, d))
        self.rho0 = np.full(n, 7850.0)
        self.mass = self.rho0 * vol
        self.movable = ~constrained
        self.left = constrained & (pos[:, 0] < 0)
        self.right = constrained & (pos[:, 0] > 0)
        self.matp = O.material_vector(80.1938e9, 164.21e9, 450e6, 715e6, 16.93, 129.24e6)
        inv = np.where(self.movable, 1.0 / self.mass, 0.0)
        self.imi, self.imj = inv[self.nbh.pair_i], inv[self.nbh.pair_j]
        self.end_disp, self.ramp_steps, self.ramp_left = 3e-5, 20, 20

    def relax_step(self, dt, eta):
        nb, mv = self.nbh, self.movable
        self.vel[mv] += 0.5 * dt * self.acc[mv]
        if self.ramp_left > 0:                           # _apply_boundary_velocity
            vbc = self.end_disp / self.ramp_steps / dt
            self.vel[self.left] = 0.0
            self.vel[self.right] = 0.0
            self.vel[self.left, 0] = -vbc
            self.vel[self.right, 0] = vbc
        else:
            self.vel[~self.movable] = 0.0
        self.pos += dt * self.vel
        raw = np.empty_like(self.F)                       # solids.deformation_rate
        self.accel.velocity_gradient_gather(np.ascontiguousarray(self.vel), nb.indptr, nb.idx,
                                            nb.grad0, nb.vol, raw)
        self.F += dt * (raw @ nb.corr)
        if self.ramp_left > 0:
            self.ramp_left -= 1
        _, pk1, self.cp, self.alpha, _, _ = self.O.return_map(self.F, self.cp, self.alpha, self.matp)
        out = np.empty_like(self.vel)                     # solids.stress_divergence_acceleration
        self.accel.pair_tensor_divergence(np.ascontiguousarray(pk1 @ nb.corr), nb.indptr, nb.idx,
                                          nb.grad0, nb.vol, out)
        self.acc = out / self.rho0[:, None]
        self.vel[mv] += 0.5 * dt * self.acc[mv]
        self.accel.damping_sweep(self.vel, nb.pair_i, nb.pair_j, nb.pair_damp, self.imi, self.imj,
                                 nb.pair_group, eta, dt)   # stepping.apply_damping_sweep


@pytest.mark.parametrize("prefix", ["n2_", "n3_"])
def test_reference_relax_step_through_the_shim_reproduces_reference_trajectory(gold_traj, prefix):
    from paper_2309_04010_b200 import accel
    pos = gold_traj[prefix + "ref_pos"]
    con = gold_traj[prefix + "constrained"]
    dp = 0.25e-3 if pos.shape[1] == 2 else 0.5e-3
    prob = _ReferenceStep(pos, gold_traj[prefix + "vol"], con, dp, accel)
    for k in range(1, 101):
        prob.relax_step(float(gold_traj[prefix + "dt"][k - 1]), 1e4)
        if k in (1, 10, 50, 100):
            s = f"{prefix}s{k}_"
            for ours, key in ((prob.pos, "pos"), (prob.vel, "vel"), (prob.F, "F"),
                              (prob.alpha, "alpha"), (prob.cp, "cp"), (prob.acc, "accel")):
                assert rel_err(ours, gold_traj[s + key]) < 1e-10, (k, key)
    assert np.max(prob.alpha) > 0
