"""Drop-in replacement for the reference's kernel module ``mtsph/_accel.py``.

Same function names, argument order, argument meaning and in-place /
out-parameter semantics as the seven numba kernels of
/root/reference/pkg/src/mtsph/_accel.py, computed by the layer-1 C ABI of
``libmtsph_b200.so`` (include/mtsph_b200.h) on the GPU.  A maintainer
switches the reference over with

    import mtsph, paper_2309_04010_b200.accel as b200_accel
    mtsph._accel = b200_accel                       # or: sys.modules["mtsph._accel"]

(INTEGRATION.md §1).  There is no CPU fallback: without the library or a
device every call raises BackendError.  Errors come back as the
reference's exception classes.

Arrays are taken as numpy arrays in the reference's layouts (float64
fields, int64 CSR / pair indices).  Outputs are written into the caller's
array; a non-contiguous or non-float64 output is filled through a
contiguous copy, as numba would write through the view.
"""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["velocity_gradient_gather", "pair_tensor_divergence",
           "pair_tensor_divergence_mapped", "scalar_difference_flux", "damping_sweep",
           "conservative_mass_rate", "porous_stress_rhs"]


def _L():
    return _lib.load_library()


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


class _Out:
    """Contiguous float64 buffer for an output argument, copied back on exit
    when the caller's array is not already one."""

    def __init__(self, arr):
        self.arr = arr
        ok = isinstance(arr, np.ndarray) and arr.dtype == np.float64 and arr.flags.c_contiguous
        self.buf = arr if ok else np.ascontiguousarray(arr, dtype=np.float64)

    def __enter__(self):
        return self.buf

    def __exit__(self, *exc):
        if self.buf is not self.arr and exc[0] is None:
            self.arr[...] = self.buf
        return False


def _dims(indptr, field):
    return len(indptr) - 1, int(np.shape(field)[1])


def velocity_gradient_gather(src, indptr, idx, grad, vol, out):
    """_accel.py:16 -- out[a] = sum_b vol[b] (src[b] - src[a]) (x) grad_ab."""
    n, d = _dims(indptr, src)
    with _Out(out) as o:
        _lib.check(_L().mtsph_velocity_gradient_gather(
            n, d, _lib.ptr(_f(src)), _lib.ptr(_i(indptr)), _lib.ptr(_i(idx)), _lib.ptr(_f(grad)),
            _lib.ptr(_f(vol)), _lib.ptr(o)))


def pair_tensor_divergence(tens, indptr, idx, grad, vol, out):
    """_accel.py:34 -- out[a] = sum_b vol[b] (tens[a] + tens[b]) . grad_ab."""
    n, d = _dims(indptr, tens)
    with _Out(out) as o:
        _lib.check(_L().mtsph_pair_tensor_divergence(
            n, d, _lib.ptr(_f(tens)), _lib.ptr(_i(indptr)), _lib.ptr(_i(idx)), _lib.ptr(_f(grad)),
            _lib.ptr(_f(vol)), _lib.ptr(o)))


def pair_tensor_divergence_mapped(tens, amap, indptr, idx, grad, vol, out):
    """_accel.py:52 -- out[a] += sum_b vol[b] (tens[a] + tens[b]) . (amap[a] grad_ab)."""
    n, d = _dims(indptr, tens)
    with _Out(out) as o:
        _lib.check(_L().mtsph_pair_tensor_divergence_mapped(
            n, d, _lib.ptr(_f(tens)), _lib.ptr(_f(amap)), _lib.ptr(_i(indptr)), _lib.ptr(_i(idx)),
            _lib.ptr(_f(grad)), _lib.ptr(_f(vol)), _lib.ptr(o)))


def scalar_difference_flux(sat, coeff, amap, indptr, idx, vol, grad, out):
    """_accel.py:76 -- out[a] = coeff[a] sum_b vol[b] (sat[a] - sat[b]) (amap[a] grad_ab)."""
    n, d = _dims(indptr, out)
    with _Out(out) as o:
        _lib.check(_L().mtsph_scalar_difference_flux(
            n, d, _lib.ptr(_f(sat)), _lib.ptr(_f(coeff)), _lib.ptr(_f(amap)), _lib.ptr(_i(indptr)),
            _lib.ptr(_i(idx)), _lib.ptr(_f(vol)), _lib.ptr(_f(grad)), _lib.ptr(o)))


def damping_sweep(vel, pair_i, pair_j, pair_damp, inv_mass_i, inv_mass_j, group_ptr, eta, dt):
    """_accel.py:171 -- the sequential pairwise implicit damping sweep, in
    place, in the reference's exact group order (forward then reverse, half
    the step each; groups solved simultaneously)."""
    n, d = np.shape(vel)
    gp = _i(group_ptr)
    with _Out(vel) as v:
        _lib.check(_L().mtsph_damping_sweep(
            n, d, _lib.ptr(v), len(pair_i), _lib.ptr(_i(pair_i)), _lib.ptr(_i(pair_j)),
            _lib.ptr(_f(pair_damp)), _lib.ptr(_f(inv_mass_i)), _lib.ptr(_f(inv_mass_j)),
            len(gp) - 1, _lib.ptr(gp), float(eta), float(dt)))


def conservative_mass_rate(flux, amap, pair_i, pair_j, pair_grad, vol, out):
    """_accel.py:210 -- antisymmetric flux-divergence mass rate (exactly
    conservative pair form)."""
    n, d = np.shape(flux)
    with _Out(out) as o:
        _lib.check(_L().mtsph_conservative_mass_rate(
            n, d, _lib.ptr(_f(flux)), _lib.ptr(_f(amap)), len(pair_i), _lib.ptr(_i(pair_i)),
            _lib.ptr(_i(pair_j)), _lib.ptr(_f(pair_grad)), _lib.ptr(_f(vol)), _lib.ptr(o)))


def porous_stress_rhs(def_grad, pressure, corr, indptr, idx, grad0, vol0, mu, lam, tbuf,
                      out_j, out_rate):
    """_accel.py:240 -- fused mixture stress -> corrected tensor T = J sigma
    F^-T B (tbuf) -> pair sum out_rate[a] = sum_b V0_b (T_a + T_b) . grad W;
    out_j = det F (rows with det F <= 0 zeroed, as the reference)."""
    n, d = _dims(indptr, def_grad)
    with _Out(tbuf) as t, _Out(out_j) as j, _Out(out_rate) as r:
        _lib.check(_L().mtsph_porous_stress_rhs(
            n, d, _lib.ptr(_f(def_grad)), _lib.ptr(_f(pressure)), _lib.ptr(_f(corr)),
            _lib.ptr(_i(indptr)), _lib.ptr(_i(idx)), _lib.ptr(_f(grad0)), _lib.ptr(_f(vol0)),
            float(mu), float(lam), _lib.ptr(t), _lib.ptr(j), _lib.ptr(r)))
