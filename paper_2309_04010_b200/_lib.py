"""ctypes binding of libmtsph_b200.so (include/mtsph_b200.h).

The product path has no CPU fallback: if the shared library is missing or
no CUDA device is visible, loading fails loudly with an explanation.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import errors

HERE = os.path.dirname(os.path.abspath(__file__))
# MTSPH_LIB: an alternative build of the same library (tuning variants,
# e.g. a different compile-time sweep ring depth); default the in-tree one
LIB_PATH = os.environ.get("MTSPH_LIB") or os.path.join(HERE, "libmtsph_b200.so")

c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_int = ctypes.c_int
c_vp = ctypes.c_void_p

SWEEP_NONE, SWEEP_SERIAL, SWEEP_COLOURED, SWEEP_TILED = 0, 1, 2, 3
SWEEPS = {"none": SWEEP_NONE, "serial": SWEEP_SERIAL, "coloured": SWEEP_COLOURED,
          "colored": SWEEP_COLOURED, "tiled": SWEEP_TILED}


class SolidDesc(ctypes.Structure):
    _fields_ = [("n", c_i64), ("d", c_int), ("pos", c_vp), ("vol", c_vp), ("rho0", c_vp),
                ("constrained", c_vp), ("side", c_vp), ("mid_mask", c_vp),
                ("h_axes", c_dbl * 3), ("shear_modulus", c_dbl), ("bulk_modulus", c_dbl),
                ("plastic", c_int), ("hardening_law", c_int), ("hard", c_dbl * 4),
                ("rm_tol", c_dbl), ("rm_max_iter", c_int), ("sweep", c_int),
                ("ghost", c_vp), ("grid", c_vp), ("tile", c_int)]


class PorousDesc(ctypes.Structure):
    _fields_ = [("n", c_i64), ("d", c_int), ("pos", c_vp), ("vol", c_vp),
                ("constrained", c_vp), ("contact", c_vp), ("h_axes", c_dbl * 3),
                ("density0", c_dbl), ("diffusivity", c_dbl), ("pressure_coeff", c_dbl),
                ("shear_modulus", c_dbl), ("lame_lambda", c_dbl), ("bulk_modulus", c_dbl),
                ("porosity", c_dbl), ("fluid_density0", c_dbl), ("initial_saturation", c_dbl),
                ("contact_time", c_dbl), ("evaporation_rate", c_dbl), ("sweep", c_int),
                ("ghost", c_vp), ("grid", c_vp), ("tile", c_int)]


class InnerParams(ctypes.Structure):
    _fields_ = [("eta", c_dbl), ("cfl", c_dbl), ("criterion", c_dbl), ("dt_outer", c_dbl),
                ("max_inner", c_i64), ("min_inner", c_i64)]


class InnerResult(ctypes.Structure):
    _fields_ = [("n_inner", c_i64), ("cap_hit", c_int), ("ek", c_dbl), ("min_dt", c_dbl),
                ("last_dt", c_dbl)]


# exported symbols (name -> (restype, argtypes)); tests check every one of
# these exists, and that the set matches include/mtsph_b200.h
SIGNATURES = {
    "mtsph_abi_version": (c_int, []),
    "mtsph_last_error": (ctypes.c_char_p, []),
    "mtsph_last_error_ids": (c_i64, [c_vp, c_i64]),
    "mtsph_device_count": (c_int, []),
    "mtsph_velocity_gradient_gather": (c_int, [c_i64, c_int] + [c_vp] * 6),
    "mtsph_pair_tensor_divergence": (c_int, [c_i64, c_int] + [c_vp] * 6),
    "mtsph_pair_tensor_divergence_mapped": (c_int, [c_i64, c_int] + [c_vp] * 7),
    "mtsph_scalar_difference_flux": (c_int, [c_i64, c_int] + [c_vp] * 8),
    "mtsph_damping_sweep": (c_int, [c_i64, c_int, c_vp, c_i64] + [c_vp] * 5
                            + [c_i64, c_vp, c_dbl, c_dbl]),
    "mtsph_conservative_mass_rate": (c_int, [c_i64, c_int, c_vp, c_vp, c_i64] + [c_vp] * 5),
    "mtsph_porous_stress_rhs": (c_int, [c_i64, c_int] + [c_vp] * 7 + [c_dbl, c_dbl]
                                + [c_vp] * 3),
    "mtsph_nbh_create": (c_int, [c_i64, c_int, c_vp, c_vp, c_vp, c_int, c_vp]),
    "mtsph_nbh_destroy": (c_int, [c_vp]),
    "mtsph_nbh_sizes": (c_int, [c_vp] * 5),
    "mtsph_nbh_export": (c_int, [c_vp] * 10),
    "mtsph_nbh_permutation": (c_int, [c_vp, c_vp]),
    "mtsph_solid_create": (c_int, [c_vp, c_vp]),
    "mtsph_solid_destroy": (c_int, [c_vp]),
    "mtsph_solid_set_ramp": (c_int, [c_vp, c_dbl, c_i64, c_i64]),
    "mtsph_solid_ramp_left": (c_int, [c_vp, c_vp]),
    "mtsph_solid_stable_dt": (c_int, [c_vp, c_dbl, c_vp]),
    "mtsph_solid_relax_step": (c_int, [c_vp, c_dbl, c_dbl, c_vp]),
    "mtsph_solid_relax": (c_int, [c_vp, c_vp, c_vp]),
    "mtsph_solid_run_steps": (c_int, [c_vp, c_vp, c_i64, c_vp]),
    "mtsph_solid_set_step": (c_int, [c_vp, c_dbl, c_dbl]),
    "mtsph_solid_phase": (c_int, [c_vp, c_int, c_int, c_vp]),
    "mtsph_solid_colours": (c_int, [c_vp, c_vp]),
    "mtsph_solid_pack": (c_int, [c_vp, ctypes.c_char_p, c_i64, c_vp, c_vp]),
    "mtsph_solid_unpack": (c_int, [c_vp, ctypes.c_char_p, c_i64, c_vp, c_vp]),
    "mtsph_solid_internal_ids": (c_int, [c_vp, c_i64, c_vp, c_vp]),
    "mtsph_solid_stream": (c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "mtsph_solid_pack_device": (c_int, [c_vp, ctypes.c_char_p, c_i64, c_vp, c_vp]),
    "mtsph_solid_unpack_device": (c_int, [c_vp, ctypes.c_char_p, c_i64, c_vp, c_vp]),
    "mtsph_solid_measure": (c_int, [c_vp, c_vp]),
    "mtsph_solid_get": (c_int, [c_vp, ctypes.c_char_p, c_vp]),
    "mtsph_solid_set": (c_int, [c_vp, ctypes.c_char_p, c_vp]),
    "mtsph_solid_launches": (c_int, [c_vp, c_vp]),
    "mtsph_solid_sizes": (c_int, [c_vp, c_vp]),
    "mtsph_solid_set_precision": (c_int, [c_vp, c_int]),
    "mtsph_porous_outer_ms": (c_int, [c_vp, c_vp]),
    "mtsph_set_device": (c_int, [c_int]),
    "mtsph_solid_phase_async": (c_int, [c_vp, c_int, c_int]),
    "mtsph_solid_begin_loop": (c_int, [c_vp, c_vp]),
    "mtsph_solid_rank_partials": (c_int, [c_vp, c_int, c_vp]),
    "mtsph_solid_control_ranks": (c_int, [c_vp, c_vp, c_int, c_int]),
    "mtsph_solid_loop_state": (c_int, [c_vp, c_vp, c_vp]),
    "mtsph_porous_sizes": (c_int, [c_vp, c_vp]),
    "mtsph_porous_set_step": (c_int, [c_vp, c_dbl, c_dbl]),
    "mtsph_porous_set_outer": (c_int, [c_vp, c_dbl, c_dbl]),
    "mtsph_porous_phase": (c_int, [c_vp, c_int, c_int, c_vp]),
    "mtsph_porous_pack": (c_int, [c_vp, ctypes.c_char_p, c_i64, c_vp, c_vp]),
    "mtsph_porous_unpack": (c_int, [c_vp, ctypes.c_char_p, c_i64, c_vp, c_vp]),
    "mtsph_porous_colours": (c_int, [c_vp, c_vp]),
    "mtsph_porous_phase_async": (c_int, [c_vp, c_int, c_int]),
    "mtsph_porous_begin_loop": (c_int, [c_vp, c_vp, c_dbl]),
    "mtsph_porous_rank_partials": (c_int, [c_vp, c_int, c_vp]),
    "mtsph_porous_control_ranks": (c_int, [c_vp, c_vp, c_int, c_int]),
    "mtsph_porous_loop_state": (c_int, [c_vp, c_vp, c_vp]),
    "mtsph_porous_internal_ids": (c_int, [c_vp, c_i64, c_vp, c_vp]),
    "mtsph_porous_stream": (c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "mtsph_porous_pack_device": (c_int, [c_vp, ctypes.c_char_p, c_i64, c_vp, c_vp]),
    "mtsph_porous_unpack_device": (c_int, [c_vp, ctypes.c_char_p, c_i64, c_vp, c_vp]),
    "mtsph_solid_precision": (c_int, [c_vp, c_vp]),
    "mtsph_porous_create": (c_int, [c_vp, c_vp]),
    "mtsph_porous_destroy": (c_int, [c_vp]),
    "mtsph_porous_advance_slow": (c_int, [c_vp, c_dbl, c_dbl, c_vp]),
    "mtsph_porous_stable_dt": (c_int, [c_vp, c_dbl, c_vp]),
    "mtsph_porous_relax_step": (c_int, [c_vp, c_dbl, c_dbl, c_vp]),
    "mtsph_porous_relax": (c_int, [c_vp, c_vp, c_vp]),
    "mtsph_porous_refresh_velocities": (c_int, [c_vp]),
    "mtsph_porous_get": (c_int, [c_vp, ctypes.c_char_p, c_vp]),
    "mtsph_porous_set": (c_int, [c_vp, ctypes.c_char_p, c_vp]),
    "mtsph_porous_launches": (c_int, [c_vp, c_vp]),
}

_LIB = None


def load_library(require_device: bool = True):
    """Load the shared library (no GPU needed unless require_device)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise errors.BackendError(
                f"{LIB_PATH} is missing: build it with "
                "`python -m paper_2309_04010_b200.build` (nvcc, sm_100a). "
                "There is no CPU fallback.")
        lib = ctypes.CDLL(LIB_PATH)
        missing = [name for name in SIGNATURES if not hasattr(lib, name)]
        if missing:
            raise errors.BackendError(f"{LIB_PATH} lacks symbols {missing}; rebuild it")
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    if require_device and _LIB.mtsph_device_count() <= 0:
        raise errors.BackendError(
            "no CUDA device visible: the mtsph B200 path runs on the GPU only "
            "(no CPU fallback)")
    return _LIB


def ptr(a):
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("arrays passed to the library must be C-contiguous")
    return a.ctypes.data_as(c_vp)


def check(status: int):
    """Translate a non-zero status into the reference's exception classes."""
    if status == 0:
        return
    lib = _LIB
    msg = lib.mtsph_last_error().decode(errors="replace")
    cnt = lib.mtsph_last_error_ids(None, 0)
    ids = np.zeros(max(cnt, 1), dtype=np.int64)
    lib.mtsph_last_error_ids(ptr(ids), cnt)
    ids = ids[:cnt].tolist()
    if status == 3:
        raise errors.GeometryError(msg)
    if status == 4:
        raise errors.SingularMomentMatrixError(ids, [0.0] * len(ids))
    if status == 5:
        raise errors.ElementInversionError(ids)
    if status == 6:
        raise errors.ReturnMapError(ids, [float("nan")] * len(ids))
    if status == 7:
        raise errors.SimulationError(msg)
    if status == 1:
        raise ValueError(msg)
    raise errors.BackendError(f"CUDA backend failure: {msg}")
