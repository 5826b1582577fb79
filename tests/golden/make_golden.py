"""Generate the golden fixtures in this directory from the REAL reference.

This script is the only place that imports the upstream `mtsph` package
(read-only checkout at /root/reference/pkg/src).  It runs in the build
container, never on the GPU box; the fixtures it writes (`*.npz`) are
committed so that tests can pin the oracle and the CUDA path without the
reference being present.

    python tests/golden/make_golden.py            # rewrites tests/golden/*.npz
    python tests/golden/make_golden.py runs       # only runs.npz (any maker name)

Every case records both the inputs and the reference outputs, so the
fixtures are self-describing.  Reference call sites used (file:line of
/root/reference/pkg/src/mtsph):
  neighbors.py:59   build_neighborhoods / neighbors.py:232 corrections
  solids.py:118     deformation_rate      solids.py:170 stress divergence
  solids.py:148     kirchhoff_stress      solids.py:164 first_pk
  plasticity.py:118 return_map
  stepping.py:101   apply_damping_sweep (-> _accel.py:171 damping_sweep)
  porous.py:141/168/194/239/266 diffusion, stress, flux, split
  _accel.py:240     porous_stress_rhs
  scenarios.py:113  NeckingProblem.relax_step, :278 PorousProblem.relax_step
  stepping.py:158   run_outer_inner
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    if not os.path.isdir(REF_SRC):
        raise SystemExit("reference checkout not found at " + REF_SRC)
    sys.path.insert(0, REF_SRC)
    import mtsph  # noqa: F401
    return mtsph


def jittered_lattice(n_side, dim, dp=1.0, jitter=0.1, seed=0):
    rng = np.random.default_rng(seed)
    axes = [np.arange(n_side) * dp] * dim
    grid = np.meshgrid(*axes, indexing="ij")
    pos = np.column_stack([g.ravel() for g in grid]).astype(float)
    pos += jitter * dp * rng.uniform(-1.0, 1.0, size=pos.shape)
    vol = np.full(len(pos), dp ** dim)
    return pos, vol


def nbh_dict(prefix, pos, vol, nbh, corr):
    spec = nbh.spec
    return {
        f"{prefix}pos": pos, f"{prefix}vol": vol,
        f"{prefix}h": np.float64(spec.h),
        f"{prefix}aniso": np.asarray(spec.anisotropy, dtype=float),
        f"{prefix}indptr": nbh.indptr, f"{prefix}idx": nbh.idx,
        f"{prefix}r0": nbh.r0, f"{prefix}grad0": nbh.grad0,
        f"{prefix}pair_i": nbh.pair_i, f"{prefix}pair_j": nbh.pair_j,
        f"{prefix}pair_damp": nbh.pair_damp,
        f"{prefix}pair_grad": nbh.pair_grad,
        f"{prefix}pair_group": nbh.pair_group,
        f"{prefix}corr": corr,
    }


def make_neighborhoods(m):
    from mtsph.kernels import KernelSpec
    from mtsph.neighbors import build_neighborhoods, compute_correction_matrices
    from mtsph.config import resolve
    from mtsph.scenarios import build

    out = {}
    cases = [("nbh2d_", *jittered_lattice(12, 2, seed=3), 1.35, ()),
             ("nbh3d_", *jittered_lattice(7, 3, seed=4), 1.35, ()),
             ("nbh2d13_", *jittered_lattice(20, 2, dp=0.1, jitter=0.0, seed=0),
              1.3 * 0.1, ())]
    for prefix, pos, vol, h, an in cases:
        spec = KernelSpec(h=h, dim=pos.shape[1], anisotropy=an)
        nbh = build_neighborhoods(pos, vol, spec)
        out.update(nbh_dict(prefix, pos, vol, nbh, compute_correction_matrices(nbh)))
    # symmetric scenario lattices: they carry multi-pair damping groups and
    # (fsi) an anisotropic kernel
    for prefix, raw in [
            ("nbhfsi2d_", {"scenario": "fsi_2d", "length": 2e-3}),
            ("nbhneck3d_", {"scenario": "necking_3d", "length": 8e-3,
                            "radius": 2e-3, "dp": 0.5e-3, "n_outer": 4}),
            ("nbhfsi3d_", {"scenario": "fsi_3d", "length": 0.5e-3,
                           "breadth": 0.5e-3, "dp": 0.125e-3 / 4})]:
        problem, _ = build(resolve(raw).params)
        nbh = problem.nbh
        out.update(nbh_dict(prefix, problem.state.ref_pos,
                            problem.state.volume0, nbh, problem.correction))
    np.savez_compressed(os.path.join(HERE, "neighborhoods.npz"), **out)
    print("neighborhoods.npz", {k: v.shape for k, v in out.items() if k.endswith("pair_i")})


def make_operators(m):
    from mtsph import solids, stepping
    from mtsph.kernels import KernelSpec
    from mtsph.neighbors import build_neighborhoods, compute_correction_matrices
    from mtsph.solids import SolidState

    rng = np.random.default_rng(101)
    out = {}
    for prefix, (pos, vol) in [("op2d_", jittered_lattice(12, 2, seed=3)),
                               ("op3d_", jittered_lattice(7, 3, seed=4))]:
        d = pos.shape[1]
        spec = KernelSpec(h=1.35, dim=d)
        nbh = build_neighborhoods(pos, vol, spec)
        corr = compute_correction_matrices(nbh)
        vel = rng.normal(size=pos.shape)
        rate = solids.deformation_rate(vel, nbh, corr)
        state = SolidState.at_rest(pos, 7850.0, vol)
        pk1 = 1e9 * rng.normal(size=(len(pos), d, d))
        acc = solids.stress_divergence_acceleration(state, pk1, nbh, corr)
        # damping sweep: every third particle constrained
        mass = 2.0 * vol * (1.0 + 0.3 * rng.uniform(size=len(vol)))
        movable = np.ones(len(vol), dtype=bool)
        movable[::3] = False
        vd = rng.normal(size=pos.shape)
        vd_out = stepping.apply_damping_sweep(vd.copy(), mass, movable, nbh,
                                              1.0e3, 1.0e-3)
        out.update({f"{prefix}pos": pos, f"{prefix}vol": vol,
                    f"{prefix}vel": vel, f"{prefix}rate": rate,
                    f"{prefix}pk1": pk1, f"{prefix}acc": acc,
                    f"{prefix}mass": mass, f"{prefix}movable": movable,
                    f"{prefix}damp_vin": vd, f"{prefix}damp_vout": vd_out})
    # damping on the symmetric scenario lattices (multi-pair groups)
    data = np.load(os.path.join(HERE, "neighborhoods.npz"))
    for prefix in ("nbhfsi2d_", "nbhneck3d_", "nbhfsi3d_"):
        pos = data[prefix + "pos"]
        vol = data[prefix + "vol"]
        spec = KernelSpec(h=float(data[prefix + "h"]), dim=pos.shape[1],
                          anisotropy=tuple(data[prefix + "aniso"]))
        nbh = build_neighborhoods(pos, vol, spec)
        mass = 1000.0 * vol * (1.0 + 0.2 * rng.uniform(size=len(vol)))
        movable = rng.uniform(size=len(vol)) > 0.1
        vd = rng.normal(size=pos.shape)
        dt = 1e-7 if prefix != "nbhneck3d_" else 1e-6
        vd_out = stepping.apply_damping_sweep(vd.copy(), mass, movable, nbh,
                                              1.0e4, dt)
        key = "damp_" + prefix
        out.update({key + "mass": mass, key + "movable": movable,
                    key + "vin": vd, key + "vout": vd_out,
                    key + "eta": np.float64(1e4), key + "dt": np.float64(dt)})
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **out)
    print("operators.npz", len(out), "arrays")


def make_constitutive(m):
    from mtsph import solids, tensors
    from mtsph.plasticity import HardeningModel, PlasticState, return_map
    from mtsph.solids import ElasticModel

    steel = ElasticModel.from_shear_bulk(80.1938e9, 164.21e9, 7850.0)
    hard = HardeningModel(450.0e6, 715.0e6, 16.93, 129.24e6)
    rng = np.random.default_rng(202)
    out = {}
    for d, n in ((3, 400), (2, 200)):
        f = np.eye(d)[None] + 0.03 * rng.normal(size=(n, d, d))
        f *= 1.0 + 0.01 * rng.normal(size=(n, 1, 1))
        f = f[tensors.det(f) > 0.5]
        chol = np.eye(d)[None] + 0.02 * rng.normal(size=(len(f), d, d))
        cp = tensors.bar(tensors.sym(chol @ tensors.transpose(chol)))
        alpha = rng.uniform(0.0, 0.3, len(f))
        # a third of the states start from the virgin plastic state so the
        # elastic branch is exercised too
        k = len(f) // 3
        cp[:k] = np.eye(d)
        alpha[:k] = 0.0
        f[:k] = np.eye(d) + 1e-4 * rng.normal(size=(k, d, d))
        tau, pk1, new, info = return_map(f, PlasticState(cp.copy(), alpha.copy()),
                                         steel, hard)
        tau_el = solids.kirchhoff_stress(f, steel)
        pk1_el = solids.first_pk(tau_el, f)
        p = f"rm{d}d_"
        out.update({p + "F": f, p + "cp": cp, p + "alpha": alpha,
                    p + "tau": tau, p + "pk1": pk1, p + "cp_new": new.cp_inv,
                    p + "alpha_new": new.alpha, p + "plastic": info["plastic"],
                    p + "dgamma": info["dgamma"], p + "tau_el": tau_el,
                    p + "pk1_el": pk1_el})
    out["steel"] = np.array([steel.shear_modulus, steel.bulk_modulus,
                             steel.density0])
    out["hard"] = np.array([450.0e6, 715.0e6, 16.93, 129.24e6])
    np.savez_compressed(os.path.join(HERE, "constitutive.npz"), **out)
    print("constitutive.npz", len(out), "arrays")


def make_porous(m):
    from mtsph import porous, tensors, _accel
    from mtsph.kernels import KernelSpec
    from mtsph.neighbors import build_neighborhoods, compute_correction_matrices
    from mtsph.porous import MembraneModel, PorousState

    model = MembraneModel(2000.0, 1.0e-10, 3.0e6, 8.242e6, 0.2631, 0.4,
                          1000.0, 0.0)
    rng = np.random.default_rng(303)
    out = {}
    for prefix, (pos, vol) in [("p2d_", jittered_lattice(9, 2, dp=1e-5, jitter=0.05, seed=8)),
                               ("p3d_", jittered_lattice(6, 3, dp=1e-5, jitter=0.05, seed=9))]:
        d = pos.shape[1]
        nbh = build_neighborhoods(pos, vol, KernelSpec(h=1.35e-5, dim=d))
        corr = compute_correction_matrices(nbh)
        state = PorousState.at_rest(pos, vol)
        state.def_grad = np.eye(d)[None] + 0.02 * rng.normal(size=(len(vol), d, d))
        j = tensors.det(state.def_grad)
        state.fluid_mass = rng.uniform(0.0, 0.35, len(vol)) * 1000.0 * vol * j
        state.fluid_mass[rng.uniform(size=len(vol)) < 0.1] = 0.0
        sat, q = porous.update_saturation_and_flux(state, nbh, model, corr)
        state.flux = q * (1.0 + 0.1 * rng.normal(size=q.shape))
        mass, clamped = porous.update_fluid_mass(state, nbh, 50.0, model, corr)
        pressure = porous.fluid_pressure(sat, model)
        tbuf = np.zeros((len(vol), d, d))
        jout = np.zeros(len(vol))
        rate = np.zeros((len(vol), d))
        _accel.porous_stress_rhs(state.def_grad, pressure, corr, nbh.indptr,
                                 nbh.idx, nbh.grad0, nbh.volume0,
                                 model.shear_modulus, model.lame_lambda,
                                 tbuf, jout, rate)
        state.vel_fluid = 1e-3 * rng.normal(size=(len(vol), d))
        frate = porous.momentum_flux_rate(state, nbh, corr)
        state.momentum = rng.normal(size=(len(vol), d))
        v_s, v_l = porous.split_velocities(state, model)
        out.update({prefix + "pos": pos, prefix + "vol": vol,
                    prefix + "F": state.def_grad,
                    prefix + "mass_in": state.fluid_mass,
                    prefix + "sat": sat, prefix + "q": q,
                    prefix + "flux_in": state.flux,
                    prefix + "mass_out": mass,
                    prefix + "clamped": np.int64(clamped),
                    prefix + "pressure": pressure, prefix + "tbuf": tbuf,
                    prefix + "J": jout, prefix + "stress_rate": rate,
                    prefix + "vel_fluid": state.vel_fluid,
                    prefix + "flux_rate": frate,
                    prefix + "momentum": state.momentum,
                    prefix + "v_s": v_s, prefix + "v_l": v_l})
    out["model"] = np.array([2000.0, 1.0e-10, 3.0e6, 8.242e6, 0.2631, 0.4,
                             1000.0, 0.0])
    np.savez_compressed(os.path.join(HERE, "porous.npz"), **out)
    print("porous.npz", len(out), "arrays")


NECK2D_TRAJ = {"scenario": "necking_2d", "length": 8e-3, "width": 2e-3,
               "dp": 0.25e-3, "stretch_per_end": 1.2e-4, "n_outer": 4,
               "ramp_steps": 20, "eta": 1e4, "energy_pct": 0.005,
               "energy_ref": 1e-4}
NECK3D_TRAJ = {"scenario": "necking_3d", "length": 8e-3, "radius": 2e-3,
               "dp": 0.5e-3, "stretch_per_end": 1.2e-4, "n_outer": 4,
               "ramp_steps": 20, "eta": 1e4, "energy_pct": 0.005,
               "energy_ref": 1e-4}
NECK2D_RUN = {"scenario": "necking_2d", "length": 8e-3, "width": 2e-3,
              "dp": 0.5e-3, "stretch_per_end": 4e-6, "n_outer": 4,
              "ramp_steps": 3, "eta": 1e4, "energy_pct": 0.005,
              "energy_ref": 1e-4}
FSI2D_RUN = {"scenario": "fsi_2d", "length": 2e-3, "t_total": 2.4,
             "n_outer": 3, "contact_time": 0.8, "max_inner": 40}
FSI3D_RUN = {"scenario": "fsi_3d", "length": 0.5e-3, "breadth": 0.5e-3,
             "dp": 0.125e-3 / 4, "t_total": 3.0, "n_outer": 3,
             "contact_time": 1.0, "max_inner": 30, "min_inner": 5}
TRAJ_STEPS = 100
TRAJ_KEEP = (1, 2, 5, 10, 25, 50, 100)


def make_trajectories(m):
    """Per-inner-step state of the reference problems (first 100 steps)."""
    from mtsph.config import resolve
    from mtsph.scenarios import build

    out = {}
    for prefix, raw in (("n2_", NECK2D_TRAJ), ("n3_", NECK3D_TRAJ)):
        problem, policy = build(resolve(raw).params)
        st = problem.state
        out.update({prefix + "ref_pos": st.ref_pos.copy(),
                    prefix + "vol": st.volume0.copy(),
                    prefix + "constrained": st.constrained.copy()})
        dts, eks = [], []
        problem.advance_slow(1, policy.dt_outer, policy.dt_outer)
        for k in range(1, TRAJ_STEPS + 1):
            dt = problem.stable_time_step(policy.cfl)
            problem.relax_step(dt, policy.eta)
            dts.append(dt)
            eks.append(problem._ek_pre_damp)
            if k in TRAJ_KEEP:
                s = f"{prefix}s{k}_"
                out.update({s + "pos": st.pos.copy(), s + "vel": st.vel.copy(),
                            s + "F": st.def_grad.copy(),
                            s + "accel": problem._accel.copy(),
                            s + "cp": problem.plastic.cp_inv.copy(),
                            s + "alpha": problem.plastic.alpha.copy()})
        out[prefix + "dt"] = np.array(dts)
        out[prefix + "ek"] = np.array(eks)
        print(prefix, "n", st.n, "plastic particles at 100:",
              int(np.count_nonzero(problem.plastic.alpha > 0)))
    np.savez_compressed(os.path.join(HERE, "trajectories.npz"), **out)
    print("trajectories.npz", len(out), "arrays")


def make_runs(m):
    """Whole outer/inner runs through run_outer_inner (observables)."""
    from mtsph.config import resolve
    from mtsph.scenarios import build
    from mtsph.stepping import run_outer_inner

    out = {}
    for prefix, raw in (("rn2_", NECK2D_RUN), ("rf2_", FSI2D_RUN),
                        ("rf3_", FSI3D_RUN)):
        problem, policy = build(resolve(raw).params)
        obs, counters = run_outer_inner(problem, policy)
        st = problem.state
        out.update({prefix + "time": obs.time,
                    prefix + "reaction_force": obs.reaction_force,
                    prefix + "neck_disp": obs.neck_disp,
                    prefix + "amplitude": obs.amplitude,
                    prefix + "ek_ratio": obs.ek_ratio,
                    prefix + "n_inner": obs.n_inner,
                    prefix + "pos": st.pos, prefix + "F": st.def_grad,
                    prefix + "clamp": np.int64(counters.clamp_events),
                    prefix + "cap_hits": np.int64(len(counters.cap_hits))})
        if hasattr(st, "vel_solid"):
            out.update({prefix + "vel": st.vel_solid,
                        prefix + "fluid_mass": st.fluid_mass,
                        prefix + "saturation": st.saturation,
                        prefix + "flux": st.flux,
                        prefix + "pressure": st.pressure,
                        prefix + "profile": obs.extras["profile"],
                        prefix + "fluid_mass_total": obs.extras["fluid_mass_total"]})
        else:
            out.update({prefix + "vel": st.vel,
                        prefix + "alpha": problem.plastic.alpha,
                        prefix + "max_alpha": obs.extras["max_alpha"]})
        print(prefix, "n", st.n, "n_inner", obs.n_inner.tolist())
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **out)
    print("runs.npz", len(out), "arrays")


# the acceptance-suite configurations (reference tests/test_acceptance.py:246
# desk necking, :323 paper-scale FSI), first outer steps only
ACCEPT_NECK = {"scenario": "necking_2d", "dp": 12.826e-3 / 25, "n_outer": 1000}
ACCEPT_FSI = {"scenario": "fsi_2d"}
ACCEPT_STEPS = {"an2_": 12, "af2_": 125}  # necking: through mid-span yield (step 11); FSI: whole run


def make_acceptance_heads(m):
    """First outer steps of the acceptance configurations (observables and
    the final state), for parity at the reference's own acceptance sizes."""
    import dataclasses
    from mtsph.config import resolve
    from mtsph.scenarios import build
    from mtsph.stepping import run_outer_inner

    out = {}
    for prefix, raw in (("an2_", ACCEPT_NECK), ("af2_", ACCEPT_FSI)):
        problem, policy = build(resolve(raw).params)
        obs, counters = run_outer_inner(
            problem, dataclasses.replace(policy, n_outer=ACCEPT_STEPS[prefix]))
        st = problem.state
        out.update({prefix + k: getattr(obs, k) for k in
                    ("time", "reaction_force", "neck_disp", "amplitude", "ek_ratio", "n_inner")})
        out[prefix + "pos"] = st.pos
        for k, v in obs.extras.items():
            out[prefix + k] = v
        if hasattr(st, "vel_solid"):
            out.update({prefix + "vel": st.vel_solid, prefix + "fluid_mass": st.fluid_mass,
                        prefix + "saturation": st.saturation})
        else:
            out.update({prefix + "vel": st.vel, prefix + "alpha": problem.plastic.alpha})
        print(prefix, "n", st.n, "n_inner", obs.n_inner.tolist())
    np.savez_compressed(os.path.join(HERE, "acceptance_heads.npz"), **out)
    print("acceptance_heads.npz", len(out), "arrays")


MAKERS = ("neighborhoods", "operators", "constitutive", "porous", "trajectories", "runs",
          "acceptance_heads")


def main():
    """make_golden.py [name ...]: all fixtures, or only the named ones."""
    m = _import_reference()
    for name in sys.argv[1:] or MAKERS:
        globals()["make_" + name](m)


if __name__ == "__main__":
    main()
