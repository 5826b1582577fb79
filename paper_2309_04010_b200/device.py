"""Thin Python handles over the device-resident problems of the C ABI.

`DeviceSolid`  <-> mtsph_solid_*  (NeckingProblem state in HBM)
`DevicePorous` <-> mtsph_porous_* (PorousProblem state in HBM)
`DeviceNeighborhood` <-> mtsph_nbh_* (neighbors.py:59 on the GPU)

All arrays crossing this boundary are host numpy arrays in the caller's
(original) particle numbering; the library keeps its own Morton order.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import check, ptr


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def _u8(a, n):
    if a is None:
        return None
    return np.ascontiguousarray(np.broadcast_to(np.asarray(a), (n,)), dtype=np.uint8)


def _h3(h_axes):
    h = list(map(float, h_axes)) + [1.0] * (3 - len(h_axes))
    return (ctypes.c_double * 3)(*h[:3])


def select_device(ordinal):
    """Place the problems created from now on (and their streams) on GPU
    `ordinal` -- one process per GPU calls this with its local rank."""
    check(_lib.load_library().mtsph_set_device(int(ordinal)))


class DeviceNeighborhood:
    """Fixed reference neighbourhood built on the GPU."""

    def __init__(self, pos, vol, h_axes, sweep="serial"):
        lib = _lib.load_library()
        pos = _f64(pos)
        n, d = pos.shape
        self.n, self.d = n, d
        h = np.ascontiguousarray(h_axes, dtype=np.float64)
        handle = ctypes.c_void_p()
        check(lib.mtsph_nbh_create(n, d, ptr(pos), ptr(_f64(vol)), ptr(h),
                                   _lib.SWEEPS[sweep], ctypes.byref(handle)))
        self._h = handle
        self._lib = lib

    def sizes(self):
        vals = [ctypes.c_int64() for _ in range(4)]
        check(self._lib.mtsph_nbh_sizes(self._h, *[ctypes.byref(v) for v in vals]))
        return tuple(v.value for v in vals)

    def export(self):
        nnz, npairs, ngroups, _ = self.sizes()
        n, d = self.n, self.d
        out = {
            "indptr": np.zeros(n + 1, np.int64), "idx": np.zeros(nnz, np.int64),
            "grad0": np.zeros((nnz, d)), "pair_i": np.zeros(npairs, np.int64),
            "pair_j": np.zeros(npairs, np.int64), "pair_damp": np.zeros(npairs),
            "pair_grad": np.zeros((npairs, d)), "pair_group": np.zeros(ngroups + 1, np.int64),
            "corr": np.zeros((n, d, d)),
        }
        check(self._lib.mtsph_nbh_export(
            self._h, ptr(out["indptr"]), ptr(out["idx"]), ptr(out["grad0"]),
            ptr(out["pair_i"]), ptr(out["pair_j"]), ptr(out["pair_damp"]),
            ptr(out["pair_grad"]), ptr(out["pair_group"]), ptr(out["corr"])))
        return out

    def permutation(self):
        p = np.zeros(self.n, np.int64)
        check(self._lib.mtsph_nbh_permutation(self._h, ptr(p)))
        return p

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.mtsph_nbh_destroy(self._h)
            self._h = None


class DeviceSolid:
    """Device-resident total-Lagrangian solid (NeckingProblem state)."""

    FIELDS_D = {"pos", "vel", "accel", "ref_pos"}
    FIELDS_DD = {"F", "cp_inv"}

    PHASES = {"kick_drift": 1, "stress": 2, "accel": 3, "sweep": 4, "vmax": 5, "amax": 6,
              "sweep_all": 7}

    def __init__(self, pos, vol, rho0, constrained, side, mid_mask, h_axes,
                 shear_modulus, bulk_modulus, plastic=True, hardening_law=0,
                 hard=(1.0, 1.0, 1.0, 0.0), rm_tol=0.0, rm_max_iter=50, sweep="serial",
                 ghost=None, grid=None, tile=0):
        lib = _lib.load_library()
        pos = _f64(pos)
        n, d = pos.shape
        self.n, self.d = n, d
        self._keep = {
            "pos": pos, "vol": _f64(vol, (n,)),
            "rho0": _f64(np.broadcast_to(np.asarray(rho0, float), (n,))),
            "constrained": _u8(constrained, n),
            "side": np.ascontiguousarray(np.broadcast_to(np.asarray(side), (n,)), dtype=np.int8),
            "mid": _u8(mid_mask if mid_mask is not None else np.zeros(n, bool), n),
            "ghost": _u8(ghost, n) if ghost is not None else None,
            "grid": _f64(grid, (6,)) if grid is not None else None,
        }
        k = self._keep
        desc = _lib.SolidDesc(
            n, d, ptr(k["pos"]).value, ptr(k["vol"]).value, ptr(k["rho0"]).value,
            ptr(k["constrained"]).value, ptr(k["side"]).value, ptr(k["mid"]).value,
            _h3(h_axes), float(shear_modulus), float(bulk_modulus), int(bool(plastic)),
            int(hardening_law), (ctypes.c_double * 4)(*[float(v) for v in hard]),
            float(rm_tol), int(rm_max_iter), _lib.SWEEPS[sweep],
            ptr(k["ghost"]).value if k["ghost"] is not None else None,
            ptr(k["grid"]).value if k["grid"] is not None else None, int(tile))
        handle = ctypes.c_void_p()
        check(lib.mtsph_solid_create(ctypes.byref(desc), ctypes.byref(handle)))
        self._h = handle
        self._lib = lib

    # -- control -------------------------------------------------------
    def set_ramp(self, end_disp, ramp_steps, ramp_left):
        check(self._lib.mtsph_solid_set_ramp(self._h, float(end_disp), int(ramp_steps),
                                             int(ramp_left)))

    def ramp_left(self):
        v = ctypes.c_int64()
        check(self._lib.mtsph_solid_ramp_left(self._h, ctypes.byref(v)))
        return v.value

    def stable_dt(self, cfl):
        v = ctypes.c_double()
        check(self._lib.mtsph_solid_stable_dt(self._h, float(cfl), ctypes.byref(v)))
        return v.value

    def relax_step(self, dt, eta):
        v = ctypes.c_double()
        check(self._lib.mtsph_solid_relax_step(self._h, float(dt), float(eta), ctypes.byref(v)))
        return v.value

    def relax(self, eta, cfl, criterion, dt_outer, max_inner=0, min_inner=1):
        p = _lib.InnerParams(float(eta), float(cfl), float(criterion), float(dt_outer),
                             int(max_inner), int(min_inner))
        r = _lib.InnerResult()
        check(self._lib.mtsph_solid_relax(self._h, ctypes.byref(p), ctypes.byref(r)))
        return r

    def run_steps(self, nsteps, eta, cfl, dt_outer=1.0):
        """Exactly nsteps inner steps (benchmark path); returns the device
        timing dict (CUDA events captured in the graph)."""
        p = _lib.InnerParams(float(eta), float(cfl), 0.0, float(dt_outer), int(nsteps), int(nsteps))
        t = np.zeros(7)
        check(self._lib.mtsph_solid_run_steps(self._h, ctypes.byref(p), int(nsteps), ptr(t)))
        return {"total_ms": t[0], "kick_drift_ms": t[1], "stress_ms": t[2], "accel_ms": t[3],
                "sweep_ms": t[4], "reduce_ms": t[5], "launches": int(t[6])}

    def set_precision(self, bits):
        """64: the reference's fp64 state (default).  32: the fp32 variant
        (csrc/solid32.cuh) -- state converted in place, the same stepping
        calls run the single-precision kernels; get/set/measure convert."""
        check(self._lib.mtsph_solid_set_precision(self._h, int(bits)))

    def precision(self):
        v = ctypes.c_int()
        check(self._lib.mtsph_solid_precision(self._h, ctypes.byref(v)))
        return v.value

    # -- multi-rank phases ------------------------------------------------
    def set_step(self, dt, eta):
        check(self._lib.mtsph_solid_set_step(self._h, float(dt), float(eta)))

    def phase(self, name, arg=0):
        out = np.zeros(2)
        check(self._lib.mtsph_solid_phase(self._h, self.PHASES[name], int(arg), ptr(out)))
        return out

    # -- device-controlled multi-rank loop (no host sync per phase) -------
    def phase_async(self, name, arg=0):
        """Enqueue a phase on stream_handle(); reductions stay on the device."""
        check(self._lib.mtsph_solid_phase_async(self._h, self.PHASES[name], int(arg)))

    def begin_loop(self, eta, cfl, criterion, dt_outer, max_inner=0, min_inner=1):
        p = _lib.InnerParams(float(eta), float(cfl), float(criterion), float(dt_outer),
                             int(max_inner), int(min_inner))
        check(self._lib.mtsph_solid_begin_loop(self._h, ctypes.byref(p)))

    def rank_partials(self, mode, dev_ptr):
        """This rank's {sum m v^2, max |a|^2, max |v|^2, error} -> 4 doubles
        at device address dev_ptr (mode 0: initial step, 1: end of step)."""
        check(self._lib.mtsph_solid_rank_partials(self._h, int(mode), dev_ptr))

    def control_ranks(self, dev_ptr, nranks, mode):
        """Stopping rule + next step from the gathered [nranks][4] partials."""
        check(self._lib.mtsph_solid_control_ranks(self._h, dev_ptr, int(nranks), int(mode)))

    def rank_partials_host(self, mode):
        import torch
        buf = torch.zeros(4, dtype=torch.float64, device="cuda")
        self.rank_partials(mode, buf.data_ptr())
        torch.cuda.ExternalStream(self.stream_handle()).synchronize()
        return buf.cpu().numpy()

    def control_ranks_host(self, gathered, mode):
        import torch
        g = torch.from_numpy(np.ascontiguousarray(gathered, dtype=np.float64).ravel()).cuda()
        torch.cuda.current_stream().synchronize()
        self.control_ranks(g.data_ptr(), len(g) // 4, mode)
        torch.cuda.ExternalStream(self.stream_handle()).synchronize()

    def loop_state(self):
        r = _lib.InnerResult()
        done = ctypes.c_int()
        check(self._lib.mtsph_solid_loop_state(self._h, ctypes.byref(r), ctypes.byref(done)))
        return bool(done.value), r

    def colours(self):
        v = ctypes.c_int()
        check(self._lib.mtsph_solid_colours(self._h, ctypes.byref(v)))
        return v.value

    def field_width(self, field):
        """doubles per particle of an exchanged field ("vel", "T")"""
        return self.d if field == "vel" else self.d * self.d

    def pack(self, field, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        w = self.field_width(field)
        out = np.zeros((len(ids), w))
        check(self._lib.mtsph_solid_pack(self._h, field.encode(), len(ids), ptr(ids), ptr(out)))
        return out

    def unpack(self, field, ids, values):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        vals = _f64(values)
        check(self._lib.mtsph_solid_unpack(self._h, field.encode(), len(ids), ptr(ids), ptr(vals)))

    # -- device-resident exchange (no host staging) ----------------------
    def internal_ids(self, ids):
        """Original local ids -> the internal ids pack/unpack_device take."""
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.zeros(len(ids), np.int64)
        check(self._lib.mtsph_solid_internal_ids(self._h, len(ids), ptr(ids), ptr(out)))
        return out

    def stream_handle(self):
        """The cudaStream_t every kernel of this solid is enqueued on."""
        s = ctypes.c_void_p()
        check(self._lib.mtsph_solid_stream(self._h, ctypes.byref(s)))
        return s.value or 0

    def pack_device(self, field, m, ids_ptr, out_ptr):
        """Pack `field` of m particles (internal ids at device address
        ids_ptr) into the device buffer at out_ptr, on stream_handle()."""
        check(self._lib.mtsph_solid_pack_device(self._h, field.encode(), int(m), ids_ptr, out_ptr))

    def unpack_device(self, field, m, ids_ptr, in_ptr):
        check(self._lib.mtsph_solid_unpack_device(self._h, field.encode(), int(m), ids_ptr, in_ptr))

    def sizes(self):
        out = np.zeros(4, np.int64)
        check(self._lib.mtsph_solid_sizes(self._h, ptr(out)))
        return {"nnz": int(out[0]), "npairs": int(out[1]), "ngroups": int(out[2]),
                "phases": int(out[3])}

    def measure(self):
        out = np.zeros(5)
        check(self._lib.mtsph_solid_measure(self._h, ptr(out)))
        return {"reaction_force": out[0], "mid_radius": out[1], "max_alpha": out[2],
                "mid_alpha_min": out[3], "finite": bool(out[4])}

    def launches(self):
        v = ctypes.c_int64()
        check(self._lib.mtsph_solid_launches(self._h, ctypes.byref(v)))
        return v.value

    # -- fields ----------------------------------------------------------
    def _shape(self, field):
        if field in self.FIELDS_D:
            return (self.n, self.d)
        if field in self.FIELDS_DD:
            return (self.n, self.d, self.d)
        if field == "alpha":
            return (self.n,)
        raise KeyError(field)

    def get(self, field):
        out = np.zeros(self._shape(field))
        check(self._lib.mtsph_solid_get(self._h, field.encode(), ptr(out)))
        return out

    def set(self, field, value):
        arr = _f64(np.broadcast_to(np.asarray(value, float), self._shape(field)))
        check(self._lib.mtsph_solid_set(self._h, field.encode(), ptr(arr)))

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.mtsph_solid_destroy(self._h)
            self._h = None


class DevicePorous:
    """Device-resident porous membrane (PorousProblem state)."""

    FIELDS_D = {"pos", "ref_pos", "momentum", "vel_solid", "vel_fluid", "flux"}
    FIELDS_DD = {"F"}
    FIELDS_1 = {"fluid_mass", "saturation", "pressure"}

    PHASES = {"kick": 1, "stress": 2, "accel": 3, "sweep": 4, "post_step": 5, "amax": 6,
              "prep_map": 7, "flux_mass": 8, "mass": 9, "prep": 10, "flux": 11, "post": 12,
              "fluxrate": 13}
    WIDTH = {"vel": None, "T": None, "satvol": 2, "rm": None, "rf": 8, "inv_mix": 1}
    EXCHANGED = ("vel", "T", "satvol", "rm", "rf", "inv_mix")

    def __init__(self, pos, vol, constrained, contact, h_axes, model, contact_time,
                 evaporation_rate, sweep="serial", ghost=None, grid=None, tile=0):
        lib = _lib.load_library()
        pos = _f64(pos)
        n, d = pos.shape
        self.n, self.d = n, d
        self._keep = {"pos": pos, "vol": _f64(vol, (n,)), "constrained": _u8(constrained, n),
                      "contact": _u8(contact, n),
                      "ghost": _u8(ghost, n) if ghost is not None else None,
                      "grid": _f64(grid, (6,)) if grid is not None else None}
        k = self._keep
        m = model
        desc = _lib.PorousDesc(
            n, d, ptr(k["pos"]).value, ptr(k["vol"]).value, ptr(k["constrained"]).value,
            ptr(k["contact"]).value, _h3(h_axes), m.density0, m.diffusivity, m.pressure_coeff,
            m.shear_modulus, m.lame_lambda, m.bulk_modulus, m.porosity, m.fluid_density0,
            m.initial_saturation, float(contact_time), float(evaporation_rate),
            _lib.SWEEPS[sweep],
            ptr(k["ghost"]).value if k["ghost"] is not None else None,
            ptr(k["grid"]).value if k["grid"] is not None else None, int(tile))
        handle = ctypes.c_void_p()
        check(lib.mtsph_porous_create(ctypes.byref(desc), ctypes.byref(handle)))
        self._h = handle
        self._lib = lib

    def advance_slow(self, dt_outer, t):
        v = ctypes.c_int64()
        check(self._lib.mtsph_porous_advance_slow(self._h, float(dt_outer), float(t),
                                                  ctypes.byref(v)))
        return v.value

    # -- multi-rank phases (slab decomposition) -------------------------
    def set_step(self, dt, eta):
        check(self._lib.mtsph_porous_set_step(self._h, float(dt), float(eta)))

    def set_outer(self, dt_outer, t):
        check(self._lib.mtsph_porous_set_outer(self._h, float(dt_outer), float(t)))

    def phase(self, name, arg=0):
        out = np.zeros(2)
        check(self._lib.mtsph_porous_phase(self._h, self.PHASES[name], int(arg), ptr(out)))
        return out

    def colours(self):
        v = ctypes.c_int()
        check(self._lib.mtsph_porous_colours(self._h, ctypes.byref(v)))
        return v.value

    def field_width(self, field):
        """doubles per particle of an exchanged field"""
        if field == "vel":
            return self.d
        if field == "T":
            return self.d * self.d
        if field == "rm":
            return 16 if self.d == 3 else 8
        return self.WIDTH[field]

    def pack(self, field, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.zeros((len(ids), self.field_width(field)))
        check(self._lib.mtsph_porous_pack(self._h, field.encode(), len(ids), ptr(ids), ptr(out)))
        return out

    def unpack(self, field, ids, values):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        vals = _f64(values)
        check(self._lib.mtsph_porous_unpack(self._h, field.encode(), len(ids), ptr(ids), ptr(vals)))

    # -- device-resident exchange and device-controlled loop ------------
    def internal_ids(self, ids):
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        out = np.zeros(len(ids), np.int64)
        check(self._lib.mtsph_porous_internal_ids(self._h, len(ids), ptr(ids), ptr(out)))
        return out

    def stream_handle(self):
        st = ctypes.c_void_p()
        check(self._lib.mtsph_porous_stream(self._h, ctypes.byref(st)))
        return st.value or 0

    def pack_device(self, field, m, ids_ptr, out_ptr):
        check(self._lib.mtsph_porous_pack_device(self._h, field.encode(), int(m), ids_ptr, out_ptr))

    def unpack_device(self, field, m, ids_ptr, in_ptr):
        check(self._lib.mtsph_porous_unpack_device(self._h, field.encode(), int(m), ids_ptr, in_ptr))

    def phase_async(self, name, arg=0):
        check(self._lib.mtsph_porous_phase_async(self._h, self.PHASES[name], int(arg)))

    def begin_loop(self, eta, cfl, criterion, dt_outer, max_inner=0, min_inner=1, vol_movable=0.0):
        p = _lib.InnerParams(float(eta), float(cfl), float(criterion), float(dt_outer),
                             int(max_inner), int(min_inner))
        check(self._lib.mtsph_porous_begin_loop(self._h, ctypes.byref(p), float(vol_movable)))

    def rank_partials(self, mode, dev_ptr):
        check(self._lib.mtsph_porous_rank_partials(self._h, int(mode), dev_ptr))

    def control_ranks(self, dev_ptr, nranks, mode):
        check(self._lib.mtsph_porous_control_ranks(self._h, dev_ptr, int(nranks), int(mode)))

    def rank_partials_host(self, mode):
        import torch
        buf = torch.zeros(4, dtype=torch.float64, device="cuda")
        self.rank_partials(mode, buf.data_ptr())
        torch.cuda.ExternalStream(self.stream_handle()).synchronize()
        return buf.cpu().numpy()

    def control_ranks_host(self, gathered, mode):
        import torch
        g = torch.from_numpy(np.ascontiguousarray(gathered, dtype=np.float64).ravel()).cuda()
        torch.cuda.current_stream().synchronize()
        self.control_ranks(g.data_ptr(), len(g) // 4, mode)
        torch.cuda.ExternalStream(self.stream_handle()).synchronize()

    def loop_state(self):
        r = _lib.InnerResult()
        done = ctypes.c_int()
        check(self._lib.mtsph_porous_loop_state(self._h, ctypes.byref(r), ctypes.byref(done)))
        return bool(done.value), r

    def sizes(self):
        out = np.zeros(4, np.int64)
        check(self._lib.mtsph_porous_sizes(self._h, ptr(out)))
        return {"nnz": int(out[0]), "npairs": int(out[1]), "ngroups": int(out[2]),
                "phases": int(out[3])}

    def outer_ms(self):
        """Device ms of the kernels of the last advance_slow (CUDA events)."""
        v = ctypes.c_double()
        check(self._lib.mtsph_porous_outer_ms(self._h, ctypes.byref(v)))
        return v.value

    def stable_dt(self, cfl):
        v = ctypes.c_double()
        check(self._lib.mtsph_porous_stable_dt(self._h, float(cfl), ctypes.byref(v)))
        return v.value

    def relax_step(self, dt, eta):
        v = ctypes.c_double()
        check(self._lib.mtsph_porous_relax_step(self._h, float(dt), float(eta), ctypes.byref(v)))
        return v.value

    def relax(self, eta, cfl, criterion, dt_outer, max_inner=0, min_inner=1):
        p = _lib.InnerParams(float(eta), float(cfl), float(criterion), float(dt_outer),
                             int(max_inner), int(min_inner))
        r = _lib.InnerResult()
        check(self._lib.mtsph_porous_relax(self._h, ctypes.byref(p), ctypes.byref(r)))
        return r

    def refresh_velocities(self):
        check(self._lib.mtsph_porous_refresh_velocities(self._h))

    def launches(self):
        v = ctypes.c_int64()
        check(self._lib.mtsph_porous_launches(self._h, ctypes.byref(v)))
        return v.value

    def _shape(self, field):
        if field in self.FIELDS_D:
            return (self.n, self.d)
        if field in self.FIELDS_DD:
            return (self.n, self.d, self.d)
        if field in self.FIELDS_1:
            return (self.n,)
        raise KeyError(field)

    def get(self, field):
        out = np.zeros(self._shape(field))
        check(self._lib.mtsph_porous_get(self._h, field.encode(), ptr(out)))
        return out

    def set(self, field, value):
        arr = _f64(np.broadcast_to(np.asarray(value, float), self._shape(field)))
        check(self._lib.mtsph_porous_set(self._h, field.encode(), ptr(arr)))

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.mtsph_porous_destroy(self._h)
            self._h = None
