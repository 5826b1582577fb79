"""Slab decomposition for multi-GPU runs (host logic, numpy only).

Particles are binned on the GLOBAL cell grid the device uses (cells of edge
2 in the scaled space X/h = the kernel support; global lower corner), and
ranks own slabs of whole cell columns along x whose boundaries are
multiples of 4 cells, so every Morton block of the tiled sweep (edge 1, 2 or
4 cells) lies inside one rank.  A rank's local problem is its owned
particles plus GHOSTS: the other ranks' particles within one cell (one
support radius) of its slab.  Because every rank bins on the same grid and
keeps the global relative order, its Morton order, blocks, neighbour lists,
sweep pairs and greedy colouring are the global ones restricted to the
slab, so a decomposed run performs exactly the single-domain operations.

Exchange plan (per rank r, for every other rank q):
  refresh[q]  = global ids of r's ghosts owned by q (sorted); q sends the
                current values of those ids in that order
  modified[c] = ghosts of r that lie in the halo (block grown by one cell)
                of one of r's sweep blocks of colour c; after phase c they
                are sent back to their owners (no other rank -- not even
                the owner -- touches them in that phase: same-coloured
                block halos are disjoint)
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

CELL = 2.0        # cell edge in the scaled space (kernel support radius)
SLAB_ALIGN = 4    # minimum slab alignment in cells (raised to the sweep tile edge)


def scaled_grid(pos, h_axes):
    """(u = X/h per axis, global lo, global hi) exactly as the device bins."""
    u = np.asarray(pos, float) / np.asarray(h_axes, float)
    return u, u.min(axis=0), u.max(axis=0)


def cell_coords(u, lo):
    return np.floor((u - lo) * 0.5).astype(np.int64)


@dataclass
class RankPlan:
    rank: int
    local_ids: np.ndarray          # global ids of the local particles (owned then ghosts? no: sorted)
    ghost: np.ndarray              # bool per local particle
    owner: np.ndarray              # owning rank per local particle
    cell_x_range: tuple            # owned cell columns [x0, x1)
    refresh_recv: dict = field(default_factory=dict)   # q -> local indices (ghosts owned by q)
    refresh_send: dict = field(default_factory=dict)   # q -> local indices (owned, ghosts on q)
    pushback_send: dict = field(default_factory=dict)  # (colour, q) -> local indices
    pushback_recv: dict = field(default_factory=dict)  # (colour, q) -> local indices
    tile_B: int = 4                # sweep block edge the colours assume (passed to the device)


def _cuts(ncell_x, counts_per_column, nranks, align=SLAB_ALIGN):
    """Slab boundaries in cell columns: multiples of `align`, balanced
    particle counts, at least one column group per rank."""
    ngroups = -(-ncell_x // align)
    if ngroups < nranks:
        raise ValueError(f"cannot split {ncell_x} cell columns into {nranks} slabs of whole "
                         f"{align}-column groups")
    padded = np.zeros(ngroups * align)
    padded[:ncell_x] = counts_per_column
    acc = np.cumsum(padded.reshape(ngroups, align).sum(axis=1))
    cut_groups = [0]
    for r in range(1, nranks):
        g = int(np.searchsorted(acc, acc[-1] * r / nranks)) + 1
        g = max(g, cut_groups[-1] + 1)                 # non-empty slab
        g = min(g, ngroups - (nranks - r))             # leave one group per remaining rank
        cut_groups.append(g)
    cut_groups.append(ngroups)
    return np.asarray(cut_groups, np.int64) * align


def block_colour_and_halo(cells, B, d):
    """Per particle: colour of its Morton block of edge B and the block
    coordinates.  Colour = block coordinates mod P, mixed-radix with the
    highest axis most significant (P = 2 for B >= 2, 3 for single cells),
    matching tiled.cuh build_tiled."""
    bc = cells >> int(np.log2(B))
    P = 2 if B >= 2 else 3
    col = np.zeros(len(cells), np.int64)
    for k in reversed(range(d)):
        col = col * P + bc[:, k] % P
    return col, bc


def _block_keys(bc, d):
    """int64 key per block coordinate row (coordinates >= -1 after shifts)."""
    bc = np.asarray(bc, np.int64) + 2
    key = np.zeros(len(bc), np.int64)
    for k in range(d):
        key = key * (1 << 21) + bc[:, k]
    return key


def make_plans(pos, h_axes, nranks, tile_B=None, ranks=None):
    """Partition into `nranks` x-slabs; returns (plans, grid(6), owner).

    ranks: build complete plans only for these ranks (one process per GPU
    needs its own); their neighbours' lists are computed as far as the
    exchange lists need them, other entries of `plans` are None.  All
    steps are vectorised (searchsorted on the sorted local id lists), so a
    rank of a many-rank run costs O(n) numpy work."""
    pos = np.asarray(pos, float)
    n, d = pos.shape
    if tile_B is None:
        tile_B = 4 if d == 3 else 16    # the device defaults (tiled.cuh build_tiled_auto)
    if tile_B not in (1, 2, 4, 8, 16):
        raise ValueError(f"tile_B must be a power of two <= 16, got {tile_B}")
    align = max(SLAB_ALIGN, tile_B)     # every sweep block inside one slab
    u, lo, hi = scaled_grid(pos, h_axes)
    cells = cell_coords(u, lo)
    del u
    ncx = int(cells[:, 0].max()) + 1
    counts = np.bincount(cells[:, 0], minlength=ncx)
    cuts = _cuts(ncx, counts, nranks, align)
    owner = np.searchsorted(cuts, cells[:, 0], side="right") - 1
    grid = np.concatenate([np.pad(lo, (0, 3 - d)), np.pad(hi, (0, 3 - d))])
    wanted = list(range(nranks)) if ranks is None else sorted(int(r) for r in ranks)
    # slabs are >= 4 cells wide and ghosts lie within one cell: only
    # adjacent ranks exchange
    need = sorted({q for r in wanted for q in (r - 1, r, r + 1) if 0 <= q < nranks})
    plans = [None] * nranks
    for r in need:
        x0, x1 = int(cuts[r]), int(cuts[r + 1])
        local = np.flatnonzero((cells[:, 0] >= x0 - 1) & (cells[:, 0] <= x1))  # ascending ids
        plans[r] = RankPlan(r, local, owner[local] != r, owner[local], (x0, x1), tile_B=tile_B)

    def at(p, gids):
        """positions of global ids (all present) in p.local_ids"""
        return np.searchsorted(p.local_ids, gids).astype(np.int64)

    # refresh lists: ghosts of r owned by q <-> owned of q that are ghosts on r
    for r in wanted:
        p = plans[r]
        for q in (r - 1, r + 1):
            if not 0 <= q < nranks:
                continue
            mine = np.flatnonzero(p.ghost & (p.owner == q))
            if len(mine):
                p.refresh_recv[q] = mine.astype(np.int64)
            pq = plans[q]
            theirs = pq.local_ids[pq.ghost & (pq.owner == r)]
            if len(theirs):
                p.refresh_send[q] = at(p, theirs)
    # sweep push-back lists: ghosts of r inside the halo (block grown by one
    # cell) of r's blocks of colour c, per owner; needed for the wanted ranks
    # and, as receive lists, for their neighbours
    shift = int(np.log2(tile_B))
    send = {}
    for r in need:
        p = plans[r]
        loc_cells = cells[p.local_ids]
        col, bc = block_colour_and_halo(loc_cells, tile_B, d)
        gidx = np.flatnonzero(p.ghost)
        gc = loc_cells[gidx]
        owned = ~p.ghost
        for c in range(1 << d):
            sel = owned & (col == c)
            if not np.any(sel) or len(gidx) == 0:
                continue
            keys = np.unique(_block_keys(bc[sel], d))
            hit = np.zeros(len(gidx), bool)
            # candidate blocks of a ghost cell g: (g-1)>>s, g>>s, (g+1)>>s per
            # axis; g lies in the halo of block b iff b B - 1 <= g <= b B + B
            offs = np.stack(np.meshgrid(*[[-1, 0, 1]] * d, indexing="ij"), -1).reshape(-1, d)
            for o in offs:
                cand = (gc + o) >> shift
                inside = np.all((gc >= cand * tile_B - 1) & (gc <= cand * tile_B + tile_B), axis=1)
                hit |= inside & np.isin(_block_keys(cand, d), keys)
            for q in np.unique(p.owner[gidx[hit]]):
                q = int(q)
                send[(r, c, q)] = gidx[hit & (p.owner[gidx] == q)].astype(np.int64)
    for (r, c, q), idx in send.items():
        if plans[r] is not None and r in wanted:
            plans[r].pushback_send[(c, q)] = idx
        if q in wanted:
            plans[q].pushback_recv[(c, r)] = at(plans[q], plans[r].local_ids[idx])
    return plans, grid, owner
