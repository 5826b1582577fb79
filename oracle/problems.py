"""Oracle problem drivers -- TEST INFRASTRUCTURE ONLY (see oracle.py).

CPU restatements of the reference's two problem classes and its outer/
inner driver, built from raw arrays so the same inputs can be handed to
the CUDA path:

  NeckingOracle  ~ scenarios.py:41  NeckingProblem
  PorousOracle   ~ scenarios.py:171 PorousProblem
  run_outer_inner ~ stepping.py:158
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import oracle as O


class NeckingOracle:
    """Displacement-driven bar; C fused relax step (mtsph_oracle.c)."""

    def __init__(self, pos, vol, rho0, constrained, left, right, mid_mask,
                 mu, bulk, hardening, h, aniso=None, end_disp_per_outer=0.0,
                 ramp_steps=1, damping_order=None, hardening_law=0):
        pos = np.ascontiguousarray(pos, dtype=float)
        n, d = pos.shape
        self.n, self.d = n, d
        self.ref_pos = pos.copy()
        self.pos = pos.copy()
        self.vel = np.zeros((n, d))
        self.F = np.ascontiguousarray(np.broadcast_to(np.eye(d), (n, d, d)))
        self.accel = np.zeros((n, d))
        self.cp = np.ascontiguousarray(np.broadcast_to(np.eye(d), (n, d, d)))
        self.alpha = np.zeros(n)
        self.vol = np.ascontiguousarray(vol, dtype=float)
        self.rho0 = np.ascontiguousarray(np.broadcast_to(np.asarray(rho0, float), (n,)))
        self.mass = self.rho0 * self.vol
        self.constrained = np.asarray(constrained, bool)
        self.movable = np.ascontiguousarray(~self.constrained, dtype=np.uint8)
        side = np.zeros(n, dtype=np.int8)
        side[np.asarray(left, bool)] = -1
        side[np.asarray(right, bool)] = 1
        self.side = side
        self.left = np.asarray(left, bool)
        self.right = np.asarray(right, bool)
        self.mid_mask = np.asarray(mid_mask, bool)
        self.nbh = O.build_nbh(pos, vol, h, aniso)
        self.h_min = float(np.min(self.nbh.h_axes))
        self.mu, self.bulk = float(mu), float(bulk)
        self.sound = math.sqrt(self.bulk / float(self.rho0[0]))
        self.elastic_only = hardening is None
        hd = hardening if hardening is not None else (1.0, 1.0, 1.0, 0.0)
        self.matp = O.material_vector(self.mu, self.bulk, *hd, law=hardening_law)
        self.end_disp = float(end_disp_per_outer)
        self.ramp_steps = max(int(ramp_steps), 1)
        self._ramp_left = 0
        self.ek_pre = 0.0
        inv = np.where(self.movable.astype(bool), 1.0 / self.mass, 0.0)
        self.imi = np.ascontiguousarray(inv[self.nbh.pair_i])
        self.imj = np.ascontiguousarray(inv[self.nbh.pair_j])
        self.gorder = None if damping_order is None else np.ascontiguousarray(damping_order, np.int64)
        self._scratch = [np.zeros((n, d, d)) for _ in range(3)]
        self._radius0 = self._mid_radius()
        self._struct = None

    @property
    def ramp_active(self):
        return self._ramp_left > 0

    def _mid_radius(self):
        t = self.pos[self.mid_mask, 1:]
        return float(np.max(np.sqrt(np.sum(t * t, axis=1))))

    def _c_struct(self):
        class S(ctypes.Structure):
            _fields_ = [("n", ctypes.c_int64), ("d", ctypes.c_int)] + \
                [(k, ctypes.c_void_p) for k in (
                    "pos", "vel", "F", "accel", "cp", "alpha", "mass", "rho0",
                    "movable", "side", "indptr", "idx", "grad0", "vol0", "corr",
                    "pi", "pj", "gp", "gorder", "pd", "imi", "imj")] + \
                [("ngroups", ctypes.c_int64)] + \
                [(k, ctypes.c_void_p) for k in ("rate", "pk1", "tmp")]
        nb = self.nbh
        p = O._p
        s = S(self.n, self.d, p(self.pos), p(self.vel), p(self.F), p(self.accel),
              p(self.cp), p(self.alpha), p(self.mass), p(self.rho0), p(self.movable),
              p(self.side), p(nb.indptr), p(nb.idx), p(nb.grad0), p(nb.vol), p(nb.corr),
              p(nb.pair_i), p(nb.pair_j), p(nb.pair_group), p(self.gorder),
              p(nb.pair_damp), p(self.imi), p(self.imj), len(nb.pair_group) - 1,
              p(self._scratch[0]), p(self._scratch[1]), p(self._scratch[2]))
        return s

    def advance_slow(self, step, dt_outer, t):
        if self.end_disp != 0.0:
            self._ramp_left = self.ramp_steps
        return 0

    def stable_time_step(self, cfl):
        if self._struct is None:
            self._struct = self._c_struct()
        return O.lib().or_necking_stable_dt(ctypes.byref(self._struct),
                                            ctypes.c_double(self.h_min),
                                            ctypes.c_double(self.sound),
                                            ctypes.c_double(cfl))

    def relax_step(self, dt, eta):
        if self._struct is None:
            self._struct = self._c_struct()
        ramp_on = self._ramp_left > 0
        vbc = self.end_disp / self.ramp_steps / dt if ramp_on else 0.0
        err = ctypes.c_int64(-1)
        ek = O.lib().or_necking_relax_step(
            ctypes.byref(self._struct), ctypes.c_double(dt), ctypes.c_double(eta),
            ctypes.c_int(1 if ramp_on else 0), ctypes.c_double(vbc),
            O._p(self.matp), ctypes.c_int(1 if self.elastic_only else 0),
            ctypes.byref(err))
        if err.value >= 0:
            raise O.OracleError(f"return map failed at particle {err.value}")
        if ramp_on:
            self._ramp_left -= 1
        self.ek_pre = ek
        return ek

    def measure(self, t):
        fx = -float(np.sum(self.mass[self.right] * self.accel[self.right, 0]))
        return {"reaction_force": fx,
                "neck_disp": self._radius0 - self._mid_radius(),
                "max_alpha": float(np.max(self.alpha)),
                "mid_alpha_min": float(np.min(self.alpha[self.mid_mask]))}

    def velocities(self):
        return self.vel


class PorousOracle:
    """Clamped porous membrane with diffusion outer step (numpy + C)."""

    def __init__(self, pos, vol, constrained, contact_mask, model: O.Membrane,
                 h, aniso, contact_time, evaporation_rate, column_id, n_columns,
                 center_column, deflection_axis, damping_order=None):
        pos = np.ascontiguousarray(pos, dtype=float)
        n, d = pos.shape
        self.n, self.d = n, d
        self.ref_pos = pos.copy()
        self.pos = pos.copy()
        self.vol0 = np.ascontiguousarray(vol, dtype=float)
        self.F = np.ascontiguousarray(np.broadcast_to(np.eye(d), (n, d, d)))
        self.momentum = np.zeros((n, d))
        self.vel_solid = np.zeros((n, d))
        self.vel_fluid = np.zeros((n, d))
        self.fluid_mass = np.zeros(n)
        self.flux = np.zeros((n, d))
        self.saturation = np.zeros(n)
        self.pressure = np.zeros(n)
        self.constrained = np.asarray(constrained, bool)
        self.movable = ~self.constrained
        self.contact = np.asarray(contact_mask, bool)
        self.m = model
        self.nbh = O.build_nbh(pos, vol, h, aniso)
        self.h_min = float(np.min(self.nbh.h_axes))
        self.contact_time = float(contact_time)
        self.evap = float(evaporation_rate)
        self.column_id = np.asarray(column_id)
        self.n_columns = int(n_columns)
        self.center_column = int(center_column)
        self.axis = int(deflection_axis)
        self.gorder = damping_order
        self.rate = np.zeros((n, d))
        self.flux_rate = np.zeros((n, d))
        self.rho_l = np.zeros(n)
        self.j = np.ones(n)
        self.ek_pre = 0.0
        self.vol_movable = float(np.sum(self.vol0[self.movable]))
        self._refresh_mass()

    ramp_active = False

    def _refresh_mass(self):
        self.mix_mass = self.m.density0 * self.vol0 + self.fluid_mass

    def _refresh_velocities(self):
        v_s, v_l = O.split_velocities(self.F, self.fluid_mass, self.momentum,
                                      self.flux, self.vol0, self.m)
        v_s[self.constrained] = 0.0
        v_l[self.constrained] = 0.0
        self.vel_solid, self.vel_fluid = v_s, v_l

    def advance_slow(self, step, dt_outer, t):
        m = self.m
        v_solid = self.vel_solid.copy()
        sat, q = O.saturation_and_flux(self.F, self.fluid_mass, self.vol0, self.nbh, m)
        self.saturation, self.flux = sat, q
        mass, clamped = O.fluid_mass_update(self.F, self.fluid_mass, self.flux, self.vol0,
                                            self.nbh, m, dt_outer)
        j = O.det(self.F)
        vol = self.vol0 * j
        if t <= self.contact_time * (1.0 + 1e-12):
            mass[self.contact] = m.porosity * m.fluid_density0 * vol[self.contact]
        elif self.evap > 0.0:
            mass = mass * np.exp(-self.evap * dt_outer)
        self.fluid_mass = mass
        sat, q = O.saturation_and_flux(self.F, self.fluid_mass, self.vol0, self.nbh, m)
        self.saturation, self.flux = sat, q
        self.pressure = m.pressure_coeff * (sat - m.sat0)
        self._refresh_mass()
        self.rho_l = sat * m.fluid_density0
        self.j = j
        rho = m.density0 / j + self.rho_l
        self.momentum = rho[:, None] * v_solid + self.flux
        self.momentum[self.constrained] = self.flux[self.constrained]
        self._refresh_velocities()
        self.flux_rate = O.momentum_flux_rate(self.F, self.vel_fluid, self.flux,
                                              self.vol0, self.nbh)
        return clamped

    def stable_time_step(self, cfl):
        v2 = np.sum(self.vel_solid ** 2, axis=1)
        dt = self.h_min / (self.m.sound_speed + float(np.sqrt(np.max(v2, initial=0.0))))
        rho = self.mix_mass / self.vol0
        a2 = np.sum(self.rate ** 2, axis=1) / (rho * rho)
        amax = float(np.sqrt(np.max(a2[self.movable], initial=0.0)))
        if amax > 0.0:
            dt = min(dt, float(np.sqrt(self.h_min / amax)))
        return cfl * dt

    def _v_solid(self, rho):
        v = (self.momentum - self.flux) / rho[:, None]
        v[self.constrained] = 0.0
        return v

    def relax_step(self, dt, eta):
        m, c = self.m, self.constrained
        self.momentum += 0.5 * dt * self.rate
        self.momentum[c] = self.flux[c]
        v_s = self._v_solid(m.density0 / self.j + self.rho_l)
        self.pos += dt * v_s
        self.F = self.F + dt * O.deformation_rate(v_s, self.nbh)
        _, jnew, rate, bad = O.porous_stress_rhs(self.F, self.pressure, self.nbh, m)
        if bad:
            raise O.OracleError("inverted element")
        self.j = jnew
        self.rate = rate + self.flux_rate
        self.momentum += 0.5 * dt * self.rate
        self.momentum[c] = self.flux[c]
        rho = m.density0 / self.j + self.rho_l
        v_s = self._v_solid(rho)
        v2 = np.sum(v_s * v_s, axis=1)
        self.ek_pre = 0.5 * float(np.sum(self.mix_mass[self.movable] * v2[self.movable])) \
            / self.vol_movable
        v_s = O.damping_sweep(v_s, self.mix_mass, self.movable, self.nbh, eta, dt,
                              order=self.gorder)
        self.vel_solid = v_s
        self.momentum = rho[:, None] * v_s + self.flux
        self.momentum[c] = self.flux[c]
        return self.ek_pre

    def deflection_profile(self):
        disp = self.pos[:, self.axis] - self.ref_pos[:, self.axis]
        s = np.bincount(self.column_id, weights=disp, minlength=self.n_columns)
        cnt = np.bincount(self.column_id, minlength=self.n_columns)
        return s / cnt

    def measure(self, t):
        self._refresh_velocities()
        prof = self.deflection_profile()
        return {"amplitude": float(prof[self.center_column]),
                "fluid_mass_total": float(np.sum(self.fluid_mass)),
                "contact_mass_total": float(np.sum(self.fluid_mass[self.contact])),
                "max_saturation": float(np.max(self.saturation)),
                "profile": prof}

    def velocities(self):
        return self.vel_solid


def run_outer_inner(problem, dt_outer, n_outer, eta, criterion, cfl=0.6,
                    max_inner=0, min_inner=1):
    """stepping.py:158 restated; returns per-outer-step records."""
    rows = []
    for step in range(1, n_outer + 1):
        t = step * dt_outer
        problem.advance_slow(step, dt_outer, t)
        n = 0
        while True:
            n += 1
            dt = problem.stable_time_step(cfl)
            problem.relax_step(dt, eta)
            ek = problem.ek_pre
            cap = max_inner if max_inner > 0 else 10 * int(np.ceil(dt_outer / dt))
            if ek <= criterion and n >= min_inner and not problem.ramp_active:
                break
            if n >= cap:
                break
        sample = problem.measure(t)
        sample.update({"time": t, "n_inner": n, "ek": ek})
        rows.append(sample)
    return rows
