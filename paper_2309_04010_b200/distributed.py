"""Multi-GPU inner relaxation: slab decomposition with halo exchanges.

Each rank holds a device-resident local problem (its slab + one cell of
ghosts, partition.py) and runs the inner step as device phases separated by
exchanges:

  kick/drift            -> refresh ghost v
  stress (gather, F, return map, T)  -> refresh ghost T
  divergence + kick     -> allreduce(sum m v^2, max |a|^2); refresh ghost v
  damping, colours 0..C-1 then C-1..0 (tiled blocks):
      sweep colour c    -> push modified ghosts back to their owners;
                           refresh ghost v
  |v|max                -> allreduce(max)
  host: kinetic-energy criterion, ramp counter, next dt (stepping.py:369-385,
        solids.py:433 -- same formulas as the device control kernel)

Because every rank bins on the global cell grid, the decomposed run
performs the single-domain tiled operations; `LocalGroup` runs all ranks in
one process (the single-GPU emulation used by the tests), `TorchGroup` is
one process per GPU over torch.distributed (NCCL on GPUs, gloo on CPU).
Exchanges are host-staged in this version (pack -> D2H -> send -> H2D ->
unpack); moving them into NCCL calls captured in the step graph is the
next step.
"""

from __future__ import annotations

import math

import numpy as np

from .device import DeviceSolid
from .partition import make_plans


class LocalGroup:
    """All ranks of the decomposition in this process (emulation)."""

    def __init__(self, plans, devices):
        self.plans = plans
        self.devices = devices

    def refresh(self, field):
        for p in self.plans:
            for q, recv_idx in p.refresh_recv.items():
                vals = self.devices[q].pack(field, self.plans[q].refresh_send[p.rank])
                self.devices[p.rank].unpack(field, recv_idx, vals)

    def pushback(self, colour):
        for p in self.plans:
            for (c, q), idx in p.pushback_send.items():
                if c != colour:
                    continue
                vals = self.devices[p.rank].pack("vel", idx)
                self.devices[q].unpack("vel", self.plans[q].pushback_recv[(c, p.rank)], vals)

    def allsum(self, values):
        return float(sum(values))

    def allmax(self, values):
        return float(max(values))


class TorchGroup:
    """One rank per process; point-to-point exchanges and reductions through
    torch.distributed (host-staged buffers)."""

    def __init__(self, plan, device, dist, tensor_device="cpu"):
        import torch
        self.torch = torch
        self.dist = dist
        self.plans = [plan]
        self.devices = [device]
        self.tdev = tensor_device

    def _swap(self, sends, recvs, width):
        """sends: {q: np.ndarray}, recvs: {q: count} -> {q: np.ndarray}"""
        torch, dist = self.torch, self.dist
        reqs, bufs = [], {}
        for q, cnt in sorted(recvs.items()):
            bufs[q] = torch.empty((cnt, width), dtype=torch.float64, device=self.tdev)
            reqs.append(dist.irecv(bufs[q], src=q))
        for q, arr in sorted(sends.items()):
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(arr)).to(self.tdev), dst=q))
        for r in reqs:
            r.wait()
        return {q: b.cpu().numpy() for q, b in bufs.items()}

    def refresh(self, field):
        p, dev = self.plans[0], self.devices[0]
        width = dev.d if field == "vel" else dev.d * dev.d
        sends = {q: dev.pack(field, idx) for q, idx in p.refresh_send.items()}
        got = self._swap(sends, {q: len(i) for q, i in p.refresh_recv.items()}, width)
        for q, vals in got.items():
            dev.unpack(field, p.refresh_recv[q], vals)

    def pushback(self, colour):
        p, dev = self.plans[0], self.devices[0]
        sends = {q: dev.pack("vel", idx) for (c, q), idx in p.pushback_send.items() if c == colour}
        recvs = {q: len(idx) for (c, q), idx in p.pushback_recv.items() if c == colour}
        got = self._swap(sends, recvs, dev.d)
        for q, vals in got.items():
            dev.unpack("vel", p.pushback_recv[(colour, q)], vals)

    def _reduce(self, value, op):
        t = self.torch.tensor([float(value)], dtype=self.torch.float64, device=self.tdev)
        self.dist.all_reduce(t, op=op)
        return float(t.item())

    def allsum(self, values):
        return self._reduce(sum(values), self.dist.ReduceOp.SUM)

    def allmax(self, values):
        return self._reduce(max(values), self.dist.ReduceOp.MAX)


def stable_dt(h, sound, cfl, vmax2, amax2):
    """solids.py:433, evaluated like the device control kernel."""
    dt = h / (sound + math.sqrt(vmax2))
    amax = math.sqrt(amax2)
    if amax > 0.0:
        dt = min(dt, math.sqrt(h / amax))
    return cfl * dt


class DecomposedSolid:
    """A necking-type solid split into x-slabs (tiled damping sweep)."""

    def __init__(self, lat, elastic, hardening, nranks, ranks=None, group="local",
                 dist=None, tensor_device="cpu", end_disp_per_outer=0.0, ramp_steps=1):
        self.plans, self.grid, self.owner = make_plans(lat.pos, lat.h_axes, nranks)
        ranks = list(range(nranks)) if ranks is None else list(ranks)
        law, hp = hardening.device_params() if hardening is not None else (0, (1.0, 1.0, 1.0, 0.0))
        devices = {}
        for r in ranks:
            p = self.plans[r]
            ids = p.local_ids
            devices[r] = DeviceSolid(lat.pos[ids], lat.vol[ids], elastic.density0,
                                     lat.constrained[ids], lat.side[ids],
                                     lat.mid_mask[ids] if lat.mid_mask is not None else None,
                                     lat.h_axes, elastic.shear_modulus, elastic.bulk_modulus,
                                     plastic=hardening is not None, hardening_law=law, hard=hp,
                                     sweep="tiled", ghost=p.ghost, grid=self.grid,
                                     tile=p.tile_B)
        if group == "local":
            self.group = LocalGroup(self.plans, [devices[r] for r in range(nranks)])
        else:
            (r,) = ranks
            self.group = TorchGroup(self.plans[r], devices[r], dist, tensor_device)
        self.devices = self.group.devices
        self.h = float(np.min(lat.h_axes))
        self.sound = elastic.sound_speed
        self.end_disp = float(end_disp_per_outer)
        self.ramp_steps = max(int(ramp_steps), 1)
        self.ramp_left = 0
        self.ncolours = max(dev.colours() for dev in self.devices)
        self.n_global = len(lat.vol)

    # -- one inner step --------------------------------------------------
    def step(self, dt, eta):
        g = self.group
        for dev in self.devices:
            dev.set_step(dt, eta)
            dev.set_ramp(self.end_disp, self.ramp_steps, self.ramp_left)
            dev.phase("kick_drift")
        g.refresh("vel")
        for dev in self.devices:
            dev.phase("stress")
        g.refresh("T")
        parts = [dev.phase("accel") for dev in self.devices]
        ek = 0.5 * g.allsum([p[0] for p in parts])
        amax2 = g.allmax([p[1] for p in parts])
        g.refresh("vel")
        nc = self.ncolours
        for rev in (False, True):
            for q in range(nc):
                c = nc - 1 - q if rev else q
                for dev in self.devices:
                    dev.phase("sweep", c + 64 if rev else c)
                g.pushback(c)
                g.refresh("vel")
        vmax2 = g.allmax([dev.phase("vmax")[0] for dev in self.devices])
        if self.ramp_left > 0:
            self.ramp_left -= 1
        return ek, vmax2, amax2

    def initial_dt(self, cfl):
        vals = [dev.phase("amax") for dev in self.devices]
        return stable_dt(self.h, self.sound, cfl, self.group.allmax([v[0] for v in vals]),
                         self.group.allmax([v[1] for v in vals]))

    def advance_slow(self):
        if self.end_disp != 0.0:
            self.ramp_left = self.ramp_steps

    def relax(self, eta, cfl, criterion, dt_outer, max_inner=0, min_inner=1, fixed_steps=None):
        """Inner loop with the reference's stopping rule (or exactly
        `fixed_steps` steps).  Returns (n_inner, ek, cap_hit, min_dt)."""
        dt = self.initial_dt(cfl)
        n, min_dt = 0, math.inf
        while True:
            n += 1
            min_dt = min(min_dt, dt)
            ek, vmax2, amax2 = self.step(dt, eta)
            if fixed_steps is not None:
                if n >= fixed_steps:
                    return n, ek, False, min_dt
            else:
                cap = max_inner if max_inner > 0 else 10 * int(math.ceil(dt_outer / dt))
                if ek <= criterion and n >= min_inner and self.ramp_left <= 0:
                    return n, ek, False, min_dt
                if n >= cap:
                    return n, ek, True, min_dt
            dt = stable_dt(self.h, self.sound, cfl, vmax2, amax2)

    def gather(self, field):
        """Owned values of `field` in global particle order (LocalGroup only)."""
        p0 = self.devices[0]
        first = self.plans[0]
        sample = p0.get(field)
        out = np.zeros((self.n_global,) + sample.shape[1:])
        for p, dev in zip(self.plans, self.devices):
            vals = sample if p is first else dev.get(field)
            own = ~p.ghost
            out[p.local_ids[own]] = vals[own]
        return out
