"""Particle generation for the benchmark scenarios.

Restates the lattice builders of the reference (scenarios.py:27-38,
:375-443, :486-566): mirror-symmetric centred offsets (exact under
reflection), cosine taper imperfection, ghost/clamp layers, contact
regions.  Adds the BASELINE.json geometries (box bars, jittered block,
cantilever strip).  Pure numpy, one-time setup.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError


@dataclass
class Lattice:
    pos: np.ndarray
    vol: np.ndarray
    h_axes: np.ndarray
    constrained: np.ndarray
    side: np.ndarray                     # -1 pulled left end, +1 right end, 0
    mid_mask: np.ndarray | None = None
    contact: np.ndarray | None = None
    column_id: np.ndarray | None = None
    column_x: np.ndarray | None = None
    center_column: int = 0
    deflection_axis: int = 1
    cross_section: float = 1.0
    extra: dict = field(default_factory=dict)

    @property
    def n(self):
        return len(self.vol)


def centred(count: int, spacing: float) -> np.ndarray:
    """Offsets symmetric about 0, exact under mirroring."""
    return (np.arange(count) - 0.5 * (count - 1)) * spacing


def taper(xoff, depth, half_width):
    """1 - depth at the centre, smooth cosine back to 1 at |x| = half_width."""
    if depth <= 0.0:
        return np.ones_like(xoff)
    inside = np.abs(xoff) < half_width
    return 1.0 - np.where(inside, 0.5 * depth * (1.0 + np.cos(np.pi * xoff / half_width)), 0.0)


def spacing_count(extent: float, dp: float, name: str) -> int:
    count = int(round(extent / dp))
    if count < 1 or abs(count * dp - extent) > 0.005 * extent:
        raise ConfigError(f"particle spacing {dp:g} does not divide {name} {extent:g} "
                          f"within 0.5%")
    return count


def _ends(col, n_cols, layers, pull):
    left = col < layers
    right = col >= n_cols - layers
    side = np.zeros(len(col), dtype=np.int8)
    side[right] = 1
    if pull == "both":
        side[left] = -1
    return left | right, side


def bar_2d(p) -> Lattice:
    """Plane bar along x (necking_2d, bar_2d), optional central taper."""
    dp = p["dp"]
    n_cols = spacing_count(p["length"], dp, "length")
    n_rows = spacing_count(p["width"], dp, "width")
    xoff = centred(n_cols, dp)
    yoff = centred(n_rows, dp)
    s = taper(xoff, p["imperfection"], 0.5 * p["imperfection_extent"] * p["length"])
    xs = np.repeat(xoff, n_rows)
    col = np.repeat(np.arange(n_cols), n_rows)
    ys = np.tile(yoff, n_cols) * np.repeat(s, n_rows)
    vol = dp * dp * np.repeat(s, n_rows)
    constrained, side = _ends(col, n_cols, int(p["layers"]), p.get("pull", "both"))
    return Lattice(np.column_stack([xs, ys]), vol, np.array([p["h_factor"] * dp] * 2),
                   constrained, side, mid_mask=np.abs(xs) <= 0.51 * dp, column_id=col,
                   cross_section=p["width"])


def cylinder_3d(p) -> Lattice:
    """Cylindrical bar (necking_3d): even transverse count, no particle on the
    y/z mirror planes."""
    dp, radius = p["dp"], p["radius"]
    n_cols = spacing_count(p["length"], dp, "length")
    n_t = 2 * int(np.round(radius / dp))
    if 2.0 * radius / dp < 8:
        raise ConfigError("need at least 8 particles across the diameter")
    xoff = centred(n_cols, dp)
    toff = centred(n_t, dp)
    s = taper(xoff, p["imperfection"], 0.5 * p["imperfection_extent"] * p["length"])
    yy, zz = np.meshgrid(toff, toff, indexing="ij")
    keep = yy ** 2 + zz ** 2 <= radius ** 2
    ys, zs = yy[keep], zz[keep]
    m = len(ys)
    sr = np.repeat(s, m)
    pos = np.column_stack([np.repeat(xoff, m), np.tile(ys, n_cols) * sr, np.tile(zs, n_cols) * sr])
    col = np.repeat(np.arange(n_cols), m)
    constrained, side = _ends(col, n_cols, int(p["layers"]), p.get("pull", "both"))
    return Lattice(pos, dp ** 3 * sr ** 2, np.array([p["h_factor"] * dp] * 3), constrained, side,
                   mid_mask=np.abs(pos[:, 0]) <= 0.51 * dp, column_id=col,
                   cross_section=np.pi * radius ** 2)


def box_3d(p, rng=None) -> Lattice:
    """Rectangular bar / block (bar_3d, block_3d); optional seeded jitter."""
    dp = p["dp"]
    nx = spacing_count(p["length"], dp, "length")
    ny = spacing_count(p["width"], dp, "width")
    nz = spacing_count(p["breadth"], dp, "breadth")
    xo, yo, zo = centred(nx, dp), centred(ny, dp), centred(nz, dp)
    X, Y, Z = np.meshgrid(xo, yo, zo, indexing="ij")
    pos = np.column_stack([X.ravel(), Y.ravel(), Z.ravel()])
    col = np.repeat(np.arange(nx), ny * nz)
    jit = p.get("jitter", 0.0)
    if jit > 0.0:
        rng = rng if rng is not None else np.random.default_rng(int(p.get("seed", 0)))
        pos = pos + jit * dp * rng.uniform(-1.0, 1.0, size=pos.shape)
    constrained, side = _ends(col, nx, int(p["layers"]), p.get("pull", "both"))
    return Lattice(pos, np.full(len(pos), dp ** 3), np.array([p["h_factor"] * dp] * 3),
                   constrained, side, mid_mask=np.abs(np.repeat(xo, ny * nz)) <= 0.51 * dp,
                   column_id=col, cross_section=p["width"] * p["breadth"])


def beam_2d(p) -> Lattice:
    """Porous beam (fsi_2d): anisotropic spacing dp_x = ratio dp, ghost clamp
    columns beyond both ends, contact on the upper half of the centre."""
    dp = p["dp"]
    ratio = p["anisotropy"]
    dpx = ratio * dp
    n_span = spacing_count(p["length"], dpx, "length")
    n_rows = spacing_count(p["width"], dp, "width")
    lay = int(p["layers"])
    xoff = (np.arange(-lay, n_span + lay + 1) - n_span / 2.0) * dpx
    yoff = centred(n_rows, dp)
    xs = np.repeat(xoff, n_rows)
    ys = np.tile(yoff, len(xoff))
    col = np.repeat(np.arange(len(xoff)), n_rows)
    half = n_span / 2.0 * dpx
    constrained = np.abs(xs) > half * (1.0 + 1e-12)
    contact = (np.abs(xs) <= 0.5 * p["contact_frac"] * p["length"] * (1.0 + 1e-12)) & (ys > 0.0)
    return Lattice(np.column_stack([xs, ys]), np.full(len(xs), dpx * dp),
                   np.array([p["h_factor"] * dp * ratio, p["h_factor"] * dp]), constrained,
                   np.zeros(len(xs), np.int8), contact=contact, column_id=col, column_x=xoff,
                   center_column=int(np.argmin(np.abs(xoff))), deflection_axis=1)


def film_3d(p) -> Lattice:
    """Porous film (fsi_3d): four clamped edges, contact on the top face."""
    dp = p["dp"]
    ratio = p["anisotropy"]
    dxy = ratio * dp
    nx = spacing_count(p["length"], dxy, "length")
    ny = spacing_count(p["breadth"], dxy, "breadth")
    nz = spacing_count(p["thickness"], dp, "thickness")
    lay = int(p["layers"])
    xoff = (np.arange(-lay, nx + lay + 1) - nx / 2.0) * dxy
    yoff = (np.arange(-lay, ny + lay + 1) - ny / 2.0) * dxy
    zoff = centred(nz, dp)
    xs, ys, zs = (a.ravel() for a in np.meshgrid(xoff, yoff, zoff, indexing="ij"))
    colx = np.repeat(np.arange(len(xoff)), len(yoff) * nz)
    constrained = (np.abs(xs) > nx / 2.0 * dxy * (1.0 + 1e-12)) | \
        (np.abs(ys) > ny / 2.0 * dxy * (1.0 + 1e-12))
    cf = 0.5 * p["contact_frac"] * (1.0 + 1e-12)
    contact = (np.abs(xs) <= cf * p["length"]) & (np.abs(ys) <= cf * p["breadth"]) & (zs > 0.0)
    h = p["h_factor"] * dp
    return Lattice(np.column_stack([xs, ys, zs]), np.full(len(xs), dxy * dxy * dp),
                   np.array([h * ratio, h * ratio, h]), constrained, np.zeros(len(xs), np.int8),
                   contact=contact, column_id=colx, column_x=xoff,
                   center_column=int(np.argmin(np.abs(xoff))), deflection_axis=2)


def strip_2d(p) -> Lattice:
    """Cantilever strip (membrane_2d): ghost clamp columns left of x = 0,
    saturation held on the top face, amplitude measured at the tip."""
    dp = p["dp"]
    n_span = spacing_count(p["length"], dp, "length")
    n_rows = spacing_count(p["width"], dp, "width")
    lay = int(p["layers"])
    icol = np.arange(-lay, n_span + 1)
    xoff = icol * dp
    yoff = centred(n_rows, dp)
    xs = np.repeat(xoff, n_rows)
    ys = np.tile(yoff, len(xoff))
    col = np.repeat(np.arange(len(xoff)), n_rows)
    constrained = np.repeat(icol < 0, n_rows)
    top = np.isclose(ys, yoff.max())
    contact = top & ~constrained
    return Lattice(np.column_stack([xs, ys]), np.full(len(xs), dp * dp),
                   np.array([p["h_factor"] * dp] * 2), constrained, np.zeros(len(xs), np.int8),
                   contact=contact, column_id=col, column_x=xoff, center_column=len(xoff) - 1,
                   deflection_axis=1)


def plate_3d(p) -> Lattice:
    """Cantilever plate (membrane_3d, BASELINE configs[3]): the strip of
    membrane_2d extruded along y -- ghost clamp columns left of x = 0 over the
    whole breadth, saturation held on the top face (z), deflection (z)
    measured at the free edge."""
    dp = p["dp"]
    n_span = spacing_count(p["length"], dp, "length")
    ny = spacing_count(p["breadth"], dp, "breadth")
    nz = spacing_count(p["thickness"], dp, "thickness")
    lay = int(p["layers"])
    icol = np.arange(-lay, n_span + 1)
    xoff = icol * dp
    yoff = centred(ny, dp)
    zoff = centred(nz, dp)
    xs, ys, zs = (a.ravel() for a in np.meshgrid(xoff, yoff, zoff, indexing="ij"))
    col = np.repeat(np.arange(len(xoff)), ny * nz)
    constrained = np.repeat(icol < 0, ny * nz)
    contact = (zs == zoff.max()) & ~constrained
    return Lattice(np.column_stack([xs, ys, zs]), np.full(len(xs), dp ** 3),
                   np.array([p["h_factor"] * dp] * 3), constrained, np.zeros(len(xs), np.int8),
                   contact=contact, column_id=col, column_x=xoff, center_column=len(xoff) - 1,
                   deflection_axis=2)


BUILDERS = {
    "necking_2d": bar_2d, "bar_2d": bar_2d, "necking_3d": cylinder_3d, "bar_3d": box_3d,
    "block_3d": box_3d, "fsi_2d": beam_2d, "fsi_3d": film_3d, "membrane_2d": strip_2d,
    "membrane_3d": plate_3d,
}


def build_lattice(params) -> Lattice:
    name = params["scenario"]
    if name not in BUILDERS:
        raise ConfigError(f"unknown scenario {name!r}")
    return BUILDERS[name](params)


def particle_count(params) -> int:
    """Lattice size without any neighbour work (cheap)."""
    name = params["scenario"]
    p = params
    if name == "fsi_2d":
        n_span = spacing_count(p["length"], p["anisotropy"] * p["dp"], "length")
        return (n_span + 2 * int(p["layers"]) + 1) * spacing_count(p["width"], p["dp"], "width")
    if name == "fsi_3d":
        dxy = p["anisotropy"] * p["dp"]
        ghost = 2 * int(p["layers"]) + 1
        return (spacing_count(p["length"], dxy, "length") + ghost) * \
            (spacing_count(p["breadth"], dxy, "breadth") + ghost) * \
            spacing_count(p["thickness"], p["dp"], "thickness")
    if name == "membrane_3d":
        return (spacing_count(p["length"], p["dp"], "length") + int(p["layers"]) + 1) * \
            spacing_count(p["breadth"], p["dp"], "breadth") * \
            spacing_count(p["thickness"], p["dp"], "thickness")
    if name in ("bar_3d", "block_3d"):
        return spacing_count(p["length"], p["dp"], "length") * \
            spacing_count(p["width"], p["dp"], "width") * \
            spacing_count(p["breadth"], p["dp"], "breadth")
    return build_lattice(params).n
