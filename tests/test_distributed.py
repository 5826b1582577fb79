"""CPU: slab decomposition plans and the torch.distributed exchange layer
(world_size 2, gloo) of the multi-GPU inner step."""

import os
import socket

import numpy as np
import pytest

from paper_2309_04010_b200 import lattices
from paper_2309_04010_b200.config import resolve
from paper_2309_04010_b200.partition import cell_coords, make_plans, scaled_grid


def _lattice(length=0.8):
    return lattices.build_lattice(resolve({"scenario": "block_3d", "length": length,
                                           "width": 0.12, "breadth": 0.12}).params)


@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_plans_partition_and_halos(nranks):
    lat = _lattice()
    plans, grid, owner = make_plans(lat.pos, lat.h_axes, nranks)
    n = len(lat.vol)
    owned = np.concatenate([p.local_ids[~p.ghost] for p in plans])
    assert np.array_equal(np.sort(owned), np.arange(n))          # a partition
    u, lo, _ = scaled_grid(lat.pos, lat.h_axes)
    cells = cell_coords(u, lo)
    for p in plans:
        assert np.all(np.diff(p.local_ids) > 0)                  # global order kept
        x0, x1 = p.cell_x_range
        assert x0 % 4 == 0 and (x1 % 4 == 0 or p.rank == nranks - 1)
        gx = cells[p.local_ids[p.ghost], 0]
        assert np.all((gx == x0 - 1) | (gx == x1))               # one cell of ghosts
        for q, idx in p.refresh_recv.items():                    # lists pair up
            send = plans[q].refresh_send[p.rank]
            assert np.array_equal(p.local_ids[idx], plans[q].local_ids[send])
    # same-colour push-back sets of different ranks never share a particle
    for c in range(8):
        touched = [p.local_ids[idx] for p in plans for (cc, q), idx in p.pushback_send.items()
                   if cc == c]
        allt = np.concatenate(touched) if touched else np.zeros(0, int)
        assert len(allt) == len(np.unique(allt))


@pytest.mark.parametrize("d", [2, 3])
@pytest.mark.parametrize("B", [1, 2, 4])
def test_block_colours_keep_same_colour_halos_disjoint(d, B):
    """Sweep-block colouring (partition.block_colour_and_halo, the host twin
    of tiled.cuh build_tiled): blocks of one colour run concurrently, so
    their halos (block grown by one cell) must never overlap -- period 2
    per axis from an edge of 2 cells, period 3 for single-cell blocks."""
    from paper_2309_04010_b200.partition import block_colour_and_halo
    ext = 4 * B + 2
    grid = np.stack(np.meshgrid(*[np.arange(ext)] * d, indexing="ij"), -1).reshape(-1, d)
    col, bc = block_colour_and_halo(grid, B, d)
    ncol = (2 if B >= 2 else 3) ** d
    assert col.min() >= 0 and col.max() < ncol
    blocks = {}
    for c, b in zip(col, map(tuple, bc)):
        assert blocks.setdefault(b, c) == c                         # one colour per block
    keys = list(blocks)
    for i, a in enumerate(keys):
        for b in keys[i + 1:]:
            if blocks[a] != blocks[b]:
                continue
            # halos [a*B - 1, a*B + B] per axis overlap iff every axis overlaps
            overlap = all(a[k] * B - 1 <= b[k] * B + B and b[k] * B - 1 <= a[k] * B + B
                          for k in range(d))
            assert not overlap, (a, b)


def test_2d_plans_align_slabs_to_the_sweep_tile():
    lat = lattices.build_lattice(resolve({"scenario": "bar_2d", "length": 8.0, "width": 1.0,
                                          "dp": 0.05}).params)
    plans, _, _ = make_plans(lat.pos, lat.h_axes, 3)
    assert all(p.tile_B == 16 for p in plans)                    # the 2D device default
    for p in plans[:-1]:
        assert p.cell_x_range[1] % 16 == 0
    with pytest.raises(ValueError, match="power of two"):
        make_plans(lat.pos, lat.h_axes, 2, tile_B=3)


class FakeDevice:
    """Test double of DeviceSolid's pack/unpack (host arrays)."""

    def __init__(self, values, d):
        self.v = values.copy()
        self.d = d

    def field_width(self, field):
        return self.d if field == "vel" else self.d * self.d

    def pack(self, field, ids):
        return self.v[np.asarray(ids)].copy()

    def unpack(self, field, ids, vals):
        self.v[np.asarray(ids)] = vals

    # device-control double: partials encode the rank, control records input
    def rank_partials_host(self, mode):
        r = float(self.rank)
        return np.array([r + 1.0, 10.0 * r, 100.0 + r, 0.0])

    def control_ranks_host(self, gathered, mode):
        self.gathered = (np.asarray(gathered).copy(), mode)


def _worker(rank, world, port, result_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_04010_b200.distributed import TorchGroup
        lat = _lattice()
        plans, _, owner = make_plans(lat.pos, lat.h_axes, world)
        p = plans[rank]
        # global "velocity" field: particle id encoded; ghosts start stale (-1)
        glob = np.stack([np.arange(len(lat.vol), dtype=float)] * 3, axis=1)
        vals = glob[p.local_ids].copy()
        vals[p.ghost] = -1.0
        dev = FakeDevice(vals, 3)
        dev.rank = rank
        g = TorchGroup(p, dev, dist)
        g.refresh("vel")
        ok_refresh = bool(np.array_equal(dev.v, glob[p.local_ids]))
        # colour-0 sweep touched: ghosts in our colour-0 halos get +1000
        for (c, q), idx in p.pushback_send.items():
            if c == 0:
                dev.v[idx] += 1000.0
        g.pushback(0)
        g.refresh("vel")
        # every particle pushed back by someone in colour 0 must now read +1000
        mine = ~p.ghost
        expect = glob[p.local_ids].copy()
        pushed = set()
        for pl in plans:
            for (c, q), idx in pl.pushback_send.items():
                if c == 0:
                    pushed.update(pl.local_ids[idx].tolist())
        bump = np.array([gid in pushed for gid in p.local_ids])
        expect[bump] += 1000.0
        ok_push = bool(np.array_equal(dev.v[mine], expect[mine]))
        s = g.allsum([rank + 1.0])
        m = g.allmax([float(rank)])
        # device control: every rank receives all ranks' partials in rank order
        g.control(1)
        want = np.concatenate([[r + 1.0, 10.0 * r, 100.0 + r, 0.0] for r in range(world)])
        ok_ctrl = bool(np.array_equal(dev.gathered[0], want)) and dev.gathered[1] == 1
        result_q.put((rank, ok_refresh, ok_push, s, m, int(bump.sum()), ok_ctrl))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_exchange():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=240) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert [r[0] for r in res] == [0, 1]
    for rank, ok_refresh, ok_push, s, m, nbump, ok_ctrl in res:
        assert ok_refresh, rank
        assert ok_push, rank
        assert ok_ctrl, rank
        assert s == 3.0 and m == 1.0
    assert sum(r[5] for r in res) > 0


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_single_rank_plans_equal_full_plans(nranks):
    """One process per GPU builds only its own plan (ranks=[r]); it must be
    the full decomposition's plan for r, exchange lists included."""
    lat = _lattice(1.2)
    full, grid, owner = make_plans(lat.pos, lat.h_axes, nranks)
    for r in range(nranks):
        sub, g2, o2 = make_plans(lat.pos, lat.h_axes, nranks, ranks=[r])
        a, b = full[r], sub[r]
        assert np.array_equal(a.local_ids, b.local_ids) and np.array_equal(a.ghost, b.ghost)
        for name in ("refresh_recv", "refresh_send", "pushback_send", "pushback_recv"):
            da, db = getattr(a, name), getattr(b, name)
            assert sorted(da) == sorted(db), (r, name)
            for k in da:
                assert np.array_equal(da[k], db[k]), (r, name, k)
        assert np.array_equal(grid, g2) and np.array_equal(owner, o2)


def test_graphed_step_falls_back_to_eager_issue_off_device(monkeypatch):
    """distributed._GraphedStep: without a device-resident (NCCL) group the
    decomposed step is never captured -- every issue is the eager enqueue --
    and MTSPH_DECOMP_GRAPH=0 gives the same on any group."""
    from paper_2309_04010_b200.distributed import _GraphedStep

    class Group:
        on_device = False

    class Loop(_GraphedStep):
        def __init__(self, group):
            self.group = group
            self.devices = []
            self.steps = 0

        def _step_async(self):
            self.steps += 1

    loop = Loop(Group())
    for _ in range(5):
        loop._issue_step()
    assert loop.steps == 5 and loop._graph is False and loop.graph_replays == 0

    class DeviceGroup:
        on_device = True

    monkeypatch.setenv("MTSPH_DECOMP_GRAPH", "0")
    loop = Loop(DeviceGroup())
    for _ in range(3):
        loop._issue_step()
    assert loop.steps == 3 and loop._graph is False
