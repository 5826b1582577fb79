"""Benchmark scenarios as device-resident problems (drop-in driver API).

`build(params) -> (problem, policy)` mirrors the reference's
scenarios.py:605: the same parameter dictionaries (config.resolve), the
same Problem protocol (advance_slow / stable_time_step / relax_step /
energy_report / measure / velocities / ramp_active) and observables,
plus `relax_inner(policy)`, which runs a whole inner relaxation loop on
the GPU.  State lives in HBM; `problem.state.<field>` reads it back in the
original particle numbering (assignment writes it; in-place mutation of a
returned array does not).
"""

from __future__ import annotations

import numpy as np

from . import lattices, stepping
from .config import FSI_SCENARIOS
from .device import DevicePorous, DeviceSolid
from .errors import ConfigError
from .materials import ElasticModel, HardeningModel, MembraneModel


class _View:
    """Attribute view of device fields (read = download, assign = upload)."""

    _MAP: dict = {}

    def __init__(self, dev, static):
        object.__setattr__(self, "_dev", dev)
        object.__setattr__(self, "_static", static)

    def __getattr__(self, name):
        mp = type(self)._MAP
        if name in mp:
            return self._dev.get(mp[name])
        static = object.__getattribute__(self, "_static")
        if name in static:
            return static[name]
        raise AttributeError(name)

    def __setattr__(self, name, value):
        mp = type(self)._MAP
        if name in mp:
            self._dev.set(mp[name], value)
        else:
            raise AttributeError(f"{name} is read-only on the device state")

    @property
    def n(self):
        return self._static["volume0"].shape[0]

    @property
    def dim(self):
        return self._static["ref_pos"].shape[1]

    @property
    def movable(self):
        return ~self._static["constrained"]


class SolidStateView(_View):
    _MAP = {"pos": "pos", "vel": "vel", "def_grad": "F"}


class PlasticView(_View):
    _MAP = {"cp_inv": "cp_inv", "alpha": "alpha"}


class PorousStateView(_View):
    _MAP = {"pos": "pos", "def_grad": "F", "momentum": "momentum", "vel_solid": "vel_solid",
            "vel_fluid": "vel_fluid", "fluid_mass": "fluid_mass", "flux": "flux",
            "saturation": "saturation", "pressure": "pressure"}


class NeckingProblem:
    """Displacement-driven elastoplastic bar (reference scenarios.py:41)."""

    def __init__(self, lat: lattices.Lattice, elastic: ElasticModel,
                 hardening: HardeningModel | None, end_disp_per_outer: float, ramp_steps: int,
                 sweep: str = "serial", rm_tol: float = 0.0):
        law, hard = hardening.device_params() if hardening is not None else (0, (1.0, 1.0, 1.0, 0.0))
        self.dev = DeviceSolid(lat.pos, lat.vol, elastic.density0, lat.constrained, lat.side,
                               lat.mid_mask, lat.h_axes, elastic.shear_modulus,
                               elastic.bulk_modulus, plastic=hardening is not None,
                               hardening_law=law, hard=hard, rm_tol=rm_tol, sweep=sweep)
        rho0 = np.full(lat.n, elastic.density0)
        self.lattice = lat
        self.state = SolidStateView(self.dev, {
            "ref_pos": lat.pos, "volume0": lat.vol, "density0": rho0,
            "mass": rho0 * lat.vol, "constrained": lat.constrained})
        self.plastic = PlasticView(self.dev, {}) if hardening is not None else None
        self.elastic = elastic
        self.hardening = hardening
        self.left = lat.constrained & (lat.pos[:, 0] < 0)
        self.right = lat.side > 0
        self.mid_mask = lat.mid_mask
        self.cross_section = lat.cross_section
        self.h_min = float(np.min(lat.h_axes))
        self.axis = 0
        self.end_disp_per_outer = float(end_disp_per_outer)
        self.ramp_steps = max(int(ramp_steps), 1)
        self.sweep = sweep
        self._ek_pre_damp = 0.0
        self._radius0 = self.dev.measure()["mid_radius"]

    # protocol -------------------------------------------------------------
    @property
    def ramp_active(self) -> bool:
        return self.dev.ramp_left() > 0

    def advance_slow(self, step, dt_outer, t) -> int:
        if self.end_disp_per_outer != 0.0:
            self.dev.set_ramp(self.end_disp_per_outer, self.ramp_steps, self.ramp_steps)
        return 0

    def stable_time_step(self, cfl: float) -> float:
        return self.dev.stable_dt(cfl)

    def relax_step(self, dt: float, eta: float) -> None:
        self._ek_pre_damp = self.dev.relax_step(dt, eta)

    def energy_report(self, policy) -> stepping.EnergyReport:
        v = self._ek_pre_damp
        return stepping.EnergyReport(v, policy.energy_reference, policy.energy_criterion,
                                     bool(v <= policy.energy_criterion))

    def relax_inner(self, policy):
        """Whole inner loop on the device; (n, report, cap_hit, min_dt)."""
        r = self.dev.relax(policy.eta, policy.cfl, policy.energy_criterion, policy.dt_outer,
                           policy.max_inner, policy.min_inner)
        self._ek_pre_damp = r.ek
        return r.n_inner, self.energy_report(policy), bool(r.cap_hit), r.min_dt

    def measure(self, t) -> dict:
        m = self.dev.measure()
        self._finite = m["finite"]
        return {"reaction_force": m["reaction_force"], "neck_disp": self._radius0 - m["mid_radius"],
                "max_alpha": m["max_alpha"], "mid_alpha_min": m["mid_alpha_min"]}

    def all_finite(self) -> bool:
        return self.dev.measure()["finite"]

    def velocities(self):
        return self.dev.get("vel")

    @property
    def _accel(self):
        return self.dev.get("accel")


class PorousProblem:
    """Clamped porous membrane, diffusion-driven swelling (scenarios.py:171)."""

    ramp_active = False

    def __init__(self, lat: lattices.Lattice, model: MembraneModel, contact_time: float,
                 evaporation_rate: float, sweep: str = "serial"):
        self.dev = DevicePorous(lat.pos, lat.vol, lat.constrained, lat.contact, lat.h_axes, model,
                                contact_time, evaporation_rate, sweep=sweep)
        self.lattice = lat
        self.model = model
        self.state = PorousStateView(self.dev, {"ref_pos": lat.pos, "volume0": lat.vol,
                                                "constrained": lat.constrained})
        self.contact_mask = lat.contact
        self.contact_time = float(contact_time)
        self.evaporation_rate = float(evaporation_rate)
        self.column_id = lat.column_id
        self.column_x = lat.column_x
        self.n_columns = len(lat.column_x)
        self.center_column = int(lat.center_column)
        self.deflection_axis = int(lat.deflection_axis)
        self.h_min = float(np.min(lat.h_axes))
        self.sweep = sweep
        self._ek_pre_damp = 0.0
        self._counts = np.bincount(self.column_id, minlength=self.n_columns)

    def advance_slow(self, step, dt_outer, t) -> int:
        return self.dev.advance_slow(dt_outer, t)

    def stable_time_step(self, cfl):
        return self.dev.stable_dt(cfl)

    def relax_step(self, dt, eta):
        self._ek_pre_damp = self.dev.relax_step(dt, eta)

    def energy_report(self, policy):
        v = self._ek_pre_damp
        return stepping.EnergyReport(v, policy.energy_reference, policy.energy_criterion,
                                     bool(v <= policy.energy_criterion))

    def relax_inner(self, policy):
        r = self.dev.relax(policy.eta, policy.cfl, policy.energy_criterion, policy.dt_outer,
                           policy.max_inner, policy.min_inner)
        self._ek_pre_damp = r.ek
        return r.n_inner, self.energy_report(policy), bool(r.cap_hit), r.min_dt

    def deflection_profile(self):
        ax = self.deflection_axis
        disp = self.dev.get("pos")[:, ax] - self.lattice.pos[:, ax]
        return np.bincount(self.column_id, weights=disp, minlength=self.n_columns) / self._counts

    def measure(self, t):
        self.dev.refresh_velocities()
        prof = self.deflection_profile()
        mass = self.dev.get("fluid_mass")
        return {"amplitude": float(prof[self.center_column]),
                "fluid_mass_total": float(np.sum(mass)),
                "contact_mass_total": float(np.sum(mass[self.contact_mask])),
                "max_saturation": float(np.max(self.dev.get("saturation"))),
                "profile": prof}

    def velocities(self):
        return self.dev.get("vel_solid")

    def all_finite(self):
        return bool(np.all(np.isfinite(self.dev.get("vel_solid"))))


# ------------------------------------------------------------------ builders

def _necking_materials(p):
    elastic = ElasticModel.from_shear_bulk(p["shear_modulus"], p["bulk_modulus"], p["density"])
    if not p["plasticity"]:
        return elastic, None
    if p.get("hardening_law", "saturation") == "power":
        hard = HardeningModel(p["initial_flow_stress"], law="power",
                              reference_strain=p["reference_strain"],
                              exponent=p["hardening_exponent"])
    else:
        hard = HardeningModel(p["initial_flow_stress"], p["saturation_flow_stress"],
                              p["saturation_exponent"], p["hardening_coefficient"])
    return elastic, hard


def _membrane(p):
    return MembraneModel(p["density"], p["diffusivity"], p["pressure_coeff"],
                         p["youngs_modulus"], p["poisson_ratio"], p["porosity"],
                         p["fluid_density"], p["initial_saturation"])


def build_problem(params, sweep=None):
    name = params["scenario"]
    sweep = sweep or params.get("damping_sweep", "serial")
    lat = lattices.build_lattice(params)
    if name in FSI_SCENARIOS:
        return PorousProblem(lat, _membrane(params), params["contact_time"],
                             params["evaporation_rate"], sweep=sweep)
    elastic, hard = _necking_materials(params)
    return NeckingProblem(lat, elastic, hard, params["stretch_per_end"] / params["n_outer"],
                          params["ramp_steps"], sweep=sweep)


def make_policy(params, h_min) -> stepping.SteppingPolicy:
    dt_outer = params["t_total"] / params["n_outer"]
    if params["scenario"] in FSI_SCENARIOS:
        limit = stepping.diffusion_time_step(h_min, params["diffusivity"])
        if dt_outer > limit * (1.0 + 1e-9):
            raise ConfigError(f"outer step {dt_outer:g} s exceeds the diffusion stability limit "
                              f"{limit:g} s; increase n_outer")
        ref = params["pressure_coeff"] * (params["porosity"] - params["initial_saturation"])
        mode = "density"
    else:
        ref = 0.5 * params["ref_force"] * params["ref_displacement"]
        mode = "total"
    if params["energy_ref"] > 0.0:
        ref = params["energy_ref"]
    return stepping.SteppingPolicy(dt_outer=dt_outer, n_outer=params["n_outer"], eta=params["eta"],
                                   energy_criterion=params["energy_pct"] * ref,
                                   energy_reference=ref, energy_mode=mode,
                                   max_inner=params["max_inner"], min_inner=params["min_inner"],
                                   cfl=params["cfl"])


def build(params, sweep=None):
    """(problem, policy) from resolved parameters (reference scenarios.py:605)."""
    if params["scenario"] not in lattices.BUILDERS:
        raise ConfigError(f"unknown scenario {params['scenario']!r}")
    lat_h = float(np.min(lattices.build_lattice(params).h_axes)) \
        if params["scenario"] in FSI_SCENARIOS else None
    if lat_h is not None:
        make_policy(params, lat_h)      # stability check before any GPU work
    problem = build_problem(params, sweep)
    return problem, make_policy(params, problem.h_min)


particle_count = lattices.particle_count


def measure_observables(problem) -> dict:
    return problem.measure(0.0)
