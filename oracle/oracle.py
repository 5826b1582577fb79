"""CPU oracle for the multi-rate SPH hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg import this module.  It is the checker the CUDA
path is compared against, never the thing measured or shipped.

It restates the upstream algorithms (numpy for one-time setup, C via
``liboracle.so`` for the per-step particle loops, see mtsph_oracle.c).  File
references are to /root/reference/pkg/src/mtsph.  It is pinned against the
golden fixtures in tests/golden (generated from the real reference by
tests/golden/make_golden.py) by tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

SIGMA = {1: 3.0 / 4.0, 2: 7.0 / (4.0 * np.pi), 3: 21.0 / (16.0 * np.pi)}
SQ23 = math.sqrt(2.0 / 3.0)


def build_lib() -> str:
    path = os.path.join(HERE, "liboracle.so")
    src = os.path.join(HERE, "mtsph_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return path


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build_lib())
        _LIB.or_necking_relax_step.restype = ctypes.c_double
        _LIB.or_necking_stable_dt.restype = ctypes.c_double
        _LIB.or_build_pairs.restype = ctypes.c_int64
        _LIB.or_return_map.restype = ctypes.c_int64
        _LIB.or_porous_stress_rhs.restype = ctypes.c_int64
        _LIB.or_split_runs.restype = ctypes.c_int64
    return _LIB


def _p(a):
    """ctypes pointer to a C-contiguous numpy array (None passes NULL)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


# ---------------------------------------------------------------- kernel

def kernel_prefactor(h_axes) -> float:
    h_axes = np.asarray(h_axes, dtype=float)
    return SIGMA[len(h_axes)] / float(np.prod(h_axes))


def kernel_gradient(rel, h_axes):
    """Vectorised dW/d(rel) (kernels.py:110)."""
    rel = np.asarray(rel, dtype=float)
    h_axes = np.asarray(h_axes, dtype=float)
    u = rel / h_axes
    q = np.sqrt(np.sum(u * u, axis=-1))
    inside = (q > 0.0) & (q < 2.0)
    t = np.where(inside, 1.0 - 0.5 * q, 0.0)
    safe = np.where(q > 0.0, q, 1.0)
    mag = kernel_prefactor(h_axes) * (-5.0 * q * t ** 3) / safe
    return np.where(inside[..., None], mag[..., None] * (u / h_axes), 0.0)


# ------------------------------------------------------------ neighbours

@dataclass
class Nbh:
    h_axes: np.ndarray
    vol: np.ndarray
    indptr: np.ndarray
    idx: np.ndarray
    grad0: np.ndarray
    pair_i: np.ndarray
    pair_j: np.ndarray
    pair_damp: np.ndarray
    pair_grad: np.ndarray
    pair_group: np.ndarray
    corr: np.ndarray

    @property
    def n(self):
        return len(self.vol)

    @property
    def dim(self):
        return len(self.h_axes)


def all_pairs(pos, h_axes):
    pos = np.ascontiguousarray(pos, dtype=float)
    n, d = pos.shape
    h_axes = np.ascontiguousarray(h_axes, dtype=float)
    cap = max(1024, n * (60 if d < 3 else 160))
    while True:
        buf = np.empty((cap, 2), dtype=np.int64)
        npairs = lib().or_build_pairs(ctypes.c_int64(n), ctypes.c_int(d), _p(pos),
                                      _p(h_axes), ctypes.c_int64(cap), _p(buf))
        if npairs == -1:
            cap *= 2
            continue
        if npairs <= -2:
            raise OracleError(f"duplicate particle positions (id {-2 - npairs})")
        return buf[:npairs]


def order_pairs(pos, pi, pj, extra_major=()):
    """Mirror-invariant deterministic pair order + damping groups.

    Restates neighbors.py:96-119 (lexsort on |midpoint - centre| keys,
    runs of equal abs-keys split into particle-sharing components by
    neighbors.py:165).  ``extra_major`` keys (most significant last) are
    placed above the reference keys; the colour-ordered sweep uses this.
    """
    d = pos.shape[1]
    if len(pi) == 0:
        return pi, pj, np.zeros(1, dtype=np.int64)
    center = 0.5 * (pos.min(axis=0) + pos.max(axis=0))
    cmid = 0.5 * (pos[pi] + pos[pj]) - center
    ab = np.abs(cmid)
    keys = [pj, pi] + [cmid[:, k] for k in range(d - 1, -1, -1)] \
        + [ab[:, k] for k in range(d - 1, -1, -1)] + list(extra_major)
    order = np.lexsort(tuple(keys))
    pi, pj, ab = pi[order], pj[order], ab[order]
    brk = np.any(ab[1:] != ab[:-1], axis=1)
    for key in extra_major:
        ks = key[order]
        brk |= ks[1:] != ks[:-1]
    starts = np.concatenate([[0], np.flatnonzero(brk) + 1, [len(pi)]])
    sizes = np.diff(starts)
    if np.all(sizes == 1):
        return pi, pj, np.arange(len(pi) + 1, dtype=np.int64)
    # union-find per run in C (mtsph_oracle.c or_split_runs)
    starts = np.ascontiguousarray(starts, dtype=np.int64)
    pi = np.ascontiguousarray(pi, dtype=np.int64)
    pj = np.ascontiguousarray(pj, dtype=np.int64)
    out = np.empty(len(pi), dtype=np.int64)
    gs = np.empty(len(pi) + 1, dtype=np.int64)
    ng = lib().or_split_runs(ctypes.c_int64(len(starts) - 1), _p(starts), _p(pi), _p(pj),
                             _p(out), _p(gs))
    if ng < 0:
        raise OracleError("more than 64 pairs share a damping group key")
    return pi[out], pj[out], gs[:ng + 1].copy()


def build_nbh(pos, vol, h, aniso=None, check_singular=True) -> Nbh:
    """Fixed reference neighbourhood + corrections (neighbors.py:59/232)."""
    pos = np.ascontiguousarray(pos, dtype=float)
    vol = np.ascontiguousarray(vol, dtype=float)
    n, d = pos.shape
    h_axes = h * np.asarray(aniso if aniso is not None and len(aniso) else (1.0,) * d,
                            dtype=float)
    pairs = all_pairs(pos, h_axes)
    pi = pairs[:, 0].copy()
    pj = pairs[:, 1].copy()
    pi, pj, gp = order_pairs(pos, pi, pj)
    if len(gp) > 1 and np.max(np.diff(gp)) > 64:
        raise OracleError("more than 64 pairs share a damping group key")
    src = np.concatenate([pi, pj])
    dst = np.concatenate([pj, pi])
    o = np.lexsort((dst, src))
    src, dst = src[o], dst[o]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    rel = pos[dst] - pos[src]
    grad0 = kernel_gradient(rel, h_axes) if len(rel) else np.zeros((0, d))
    if len(pi):
        relp = pos[pj] - pos[pi]
        rp = np.sqrt(np.sum(relp * relp, axis=1))
        pgrad = kernel_gradient(relp, h_axes)
        radial = -np.sum((relp / rp[:, None]) * pgrad, axis=1)
        pdamp = 2.0 * vol[pi] * vol[pj] * radial / rp
    else:
        pgrad = np.zeros((0, d))
        pdamp = np.zeros(0)
    # moment matrices M_a = sum_b V_b (X_b - X_a) (x) grad_ab; the reference
    # forms X_b - X_a as |r| * (r/|r|)
    r0 = np.sqrt(np.sum(rel * rel, axis=1)) if len(rel) else np.zeros(0)
    relr = r0[:, None] * (rel / np.where(r0 > 0, r0, 1.0)[:, None]) if len(rel) else rel
    mom = np.zeros((n, d, d))
    owner = src
    np.add.at(mom, owner, vol[dst, None, None] * relr[:, :, None] * grad0[:, None, :])
    dets = np.linalg.det(mom) if n else np.zeros(0)
    scale = np.sqrt(np.sum(mom * mom, axis=(1, 2))) ** d + np.finfo(float).tiny
    bad = np.flatnonzero(np.abs(dets) <= 1e-12 * scale)
    if check_singular and bad.size:
        raise OracleError(f"singular moment matrix at particles {bad[:10].tolist()}")
    corr = np.zeros_like(mom)
    good = np.abs(dets) > 1e-12 * scale
    corr[good] = np.linalg.inv(mom[good])
    return Nbh(h_axes, vol, indptr, dst.astype(np.int64), np.ascontiguousarray(grad0),
               pi.astype(np.int64), pj.astype(np.int64), pdamp,
               np.ascontiguousarray(pgrad), gp, np.ascontiguousarray(corr))


# ------------------------------------------------------------ operators

def deformation_rate(vel, nbh: Nbh):
    n, d = vel.shape
    raw = np.empty((n, d, d))
    lib().or_velocity_gradient_gather(
        ctypes.c_int64(n), ctypes.c_int(d), _p(np.ascontiguousarray(vel)),
        _p(nbh.indptr), _p(nbh.idx), _p(nbh.grad0), _p(nbh.vol), _p(raw))
    return raw @ nbh.corr


def stress_divergence(pk1, rho0, nbh: Nbh):
    n, d = pk1.shape[:2]
    t = np.ascontiguousarray(pk1 @ nbh.corr)
    out = np.empty((n, d))
    lib().or_pair_tensor_divergence(ctypes.c_int64(n), ctypes.c_int(d), _p(t),
                                    _p(nbh.indptr), _p(nbh.idx), _p(nbh.grad0),
                                    _p(nbh.vol), _p(out))
    return out / np.broadcast_to(rho0, (n,))[:, None]


def material_vector(mu, K, s0=1.0, sinf=1.0, delta=1.0, H=0.0, tol=None, max_iter=50, law=0):
    """law 0: reference saturation+linear hardening (plasticity.py:64);
    law 1: power law s0 (1 + a/e0)^m passed as (s0, e0, m, 0)."""
    if tol is None:
        tol = 1e-8 * s0
    return np.array([mu, K, s0, sinf, delta, H, tol, float(max_iter), float(law)])


def return_map(F, cp, alpha, matp, elastic_only=False):
    """Batched return map; returns tau, pk1, cp_new, alpha_new, plastic, dgamma."""
    F = np.ascontiguousarray(F, dtype=float)
    n, d = F.shape[:2]
    cp = np.ascontiguousarray(cp, dtype=float).copy()
    alpha = np.ascontiguousarray(alpha, dtype=float).copy()
    tau = np.empty_like(F)
    pk1 = np.empty_like(F)
    plastic = np.zeros(n, dtype=np.int32)
    dg = np.zeros(n)
    st = np.zeros(1, dtype=np.int32)
    first = lib().or_return_map(ctypes.c_int64(n), ctypes.c_int(d), _p(F), _p(cp),
                                _p(alpha), _p(np.ascontiguousarray(matp, dtype=float)),
                                _p(tau), _p(pk1), _p(plastic), _p(dg),
                                ctypes.c_int(1 if elastic_only else 0), _p(st))
    if first >= 0:
        raise OracleError(f"return map failed at particle {first} (kind {st[0]})")
    return tau, pk1, cp, alpha, plastic.astype(bool), dg


def damping_sweep(vel, mass, movable, nbh: Nbh, eta, dt, order=None):
    vel = np.ascontiguousarray(vel, dtype=float)
    d = vel.shape[1]
    inv = np.where(movable, 1.0 / mass, 0.0)
    imi = np.ascontiguousarray(inv[nbh.pair_i])
    imj = np.ascontiguousarray(inv[nbh.pair_j])
    ng = len(nbh.pair_group) - 1
    lib().or_damping_sweep(ctypes.c_int(d), _p(vel), _p(nbh.pair_i), _p(nbh.pair_j),
                           _p(nbh.pair_damp), _p(imi), _p(imj), ctypes.c_int64(ng),
                           _p(nbh.pair_group),
                           _p(None if order is None else np.ascontiguousarray(order, dtype=np.int64)),
                           ctypes.c_double(eta), ctypes.c_double(dt))
    return vel


# ------------------------------------------------------------- porous

@dataclass(frozen=True)
class Membrane:
    density0: float
    diffusivity: float
    pressure_coeff: float
    youngs: float
    poisson: float
    porosity: float
    fluid_density0: float
    sat0: float

    @property
    def mu(self):
        return self.youngs / (2.0 * (1.0 + self.poisson))

    @property
    def bulk(self):
        return self.youngs / (3.0 * (1.0 - 2.0 * self.poisson))

    @property
    def lam(self):
        return self.bulk - 2.0 * self.mu / 3.0

    @property
    def sound_speed(self):
        return math.sqrt(self.bulk / self.density0)


def det(t):
    return np.linalg.det(t) if t.shape[-1] > 1 else t[..., 0, 0].copy()


def _amap(F, corr):
    return np.ascontiguousarray(np.linalg.inv(F) @ np.swapaxes(corr, -1, -2))


def saturation_and_flux(F, fluid_mass, vol0, nbh: Nbh, m: Membrane):
    """porous.py:168: saturation from mass, Fick flux down its gradient."""
    n, d = fluid_mass.shape[0], F.shape[1]
    j = det(F)
    if np.any(j <= 0):
        raise OracleError("inverted element")
    vol = np.ascontiguousarray(vol0 * j)
    rho_l = fluid_mass / vol
    sat = np.ascontiguousarray(rho_l / m.fluid_density0)
    coeff = np.ascontiguousarray(m.diffusivity * rho_l)
    q = np.empty((n, d))
    lib().or_scalar_difference_flux(ctypes.c_int64(n), ctypes.c_int(d), _p(sat), _p(coeff),
                                    _p(_amap(F, nbh.corr)), _p(nbh.indptr), _p(nbh.idx),
                                    _p(vol), _p(nbh.grad0), _p(q))
    return sat, q


def fluid_mass_update(F, fluid_mass, flux, vol0, nbh: Nbh, m: Membrane, dt):
    """porous.py:141 (conservative pair form + clamp); returns mass, clamped."""
    n, d = fluid_mass.shape[0], F.shape[1]
    j = det(F)
    vol = np.ascontiguousarray(vol0 * j)
    rate = np.empty(n)
    lib().or_conservative_mass_rate(ctypes.c_int64(n), ctypes.c_int(d),
                                    _p(np.ascontiguousarray(flux)), _p(_amap(F, nbh.corr)),
                                    ctypes.c_int64(len(nbh.pair_i)), _p(nbh.pair_i),
                                    _p(nbh.pair_j), _p(nbh.pair_grad), _p(vol), _p(rate))
    mass = fluid_mass + dt * rate
    cap = m.porosity * m.fluid_density0 * vol
    clamped = int(np.count_nonzero((mass < 0.0) | (mass > cap)))
    return np.clip(mass, 0.0, cap), clamped


def porous_stress_rhs(F, pressure, nbh: Nbh, m: Membrane):
    n, d = F.shape[:2]
    tbuf = np.empty_like(F)
    jout = np.empty(n)
    rate = np.empty((n, d))
    bad = lib().or_porous_stress_rhs(ctypes.c_int64(n), ctypes.c_int(d),
                                     _p(np.ascontiguousarray(F)),
                                     _p(np.ascontiguousarray(pressure)), _p(nbh.corr),
                                     _p(nbh.indptr), _p(nbh.idx), _p(nbh.grad0), _p(nbh.vol),
                                     ctypes.c_double(m.mu), ctypes.c_double(m.lam),
                                     _p(tbuf), _p(jout), _p(rate))
    return tbuf, jout, rate, int(bad)


def momentum_flux_rate(F, vel_fluid, flux, vol0, nbh: Nbh):
    """porous.py:239: -sum_b V_b ((vq)_a + (vq)_b) . (F_a^-1 B_a^T grad)."""
    n, d = flux.shape
    out = np.zeros((n, d))
    vq = np.ascontiguousarray(vel_fluid[:, :, None] * flux[:, None, :])
    if np.any(vq):
        j = det(F)
        amap = np.ascontiguousarray(-_amap(F, nbh.corr))
        lib().or_pair_tensor_divergence_mapped(
            ctypes.c_int64(n), ctypes.c_int(d), _p(vq), _p(amap), _p(nbh.indptr),
            _p(nbh.idx), _p(nbh.grad0), _p(np.ascontiguousarray(vol0 * j)), _p(out))
    return out


def split_velocities(F, fluid_mass, momentum, flux, vol0, m: Membrane):
    """porous.py:266 with the dry-region guard."""
    j = det(F)
    rho_s = m.density0 / j
    rho_l = fluid_mass / (vol0 * j)
    rho = rho_s + rho_l
    dry = rho_l < 1e-12 * m.fluid_density0
    fl = np.where(dry[:, None], 0.0, flux)
    v_s = (momentum - fl) / rho[:, None]
    safe = np.where(dry, 1.0, rho_l)
    v_l = np.where(dry[:, None], v_s, v_s + fl / safe[:, None])
    return v_s, v_l
