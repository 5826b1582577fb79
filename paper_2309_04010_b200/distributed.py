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
  host: kinetic-energy criterion, ramp counter, next dt (stepping.py:177-195,
        solids.py:187 -- same formulas as the device control kernel)

Because every rank bins on the global cell grid, the decomposed run
performs the single-domain tiled operations; `LocalGroup` runs all ranks in
one process (the single-GPU emulation used by the tests), `TorchGroup` is
one process per GPU over torch.distributed (NCCL on GPUs, gloo on CPU).
TorchGroup exchanges are host-staged over gloo (pack -> D2H -> send -> H2D
-> unpack) and device-resident over NCCL (pack kernel -> NCCL send/recv of
device buffers -> unpack kernel, stream-ordered on the solid's stream);
the per-phase reductions still return to the host.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from .device import DeviceSolid
from .partition import make_plans


class LocalGroup:
    """All ranks of the decomposition in this process (emulation).

    device_buffers=False: host pack/unpack.  True: the device-resident path
    of TorchGroup(tensor_device="cuda") -- internal-id lists on the device,
    pack kernel -> CUDA buffer -> unpack kernel -- with a device copy between
    the two solids' streams standing in for the NCCL send/recv."""

    def __init__(self, plans, devices, device_buffers=False):
        self.plans = plans
        self.devices = devices
        self.device_buffers = device_buffers
        self._cache = {}

    def _move(self, field, src, src_idx, dst, dst_idx):
        if not self.device_buffers:
            self.devices[dst].unpack(field, dst_idx, self.devices[src].pack(field, src_idx))
            return
        import torch
        key = (field, src, dst, id(src_idx))
        if key not in self._cache:
            s, t = self.devices[src], self.devices[dst]
            w = s.field_width(field)
            self._cache[key] = (torch.from_numpy(s.internal_ids(src_idx)).cuda(),
                                torch.from_numpy(t.internal_ids(dst_idx)).cuda(),
                                torch.empty((len(src_idx), w), dtype=torch.float64, device="cuda"))
        ids_s, ids_t, buf = self._cache[key]
        s, t = self.devices[src], self.devices[dst]
        s.pack_device(field, len(ids_s), ids_s.data_ptr(), buf.data_ptr())
        torch.cuda.ExternalStream(s.stream_handle()).synchronize()
        t.unpack_device(field, len(ids_t), ids_t.data_ptr(), buf.data_ptr())
        torch.cuda.ExternalStream(t.stream_handle()).synchronize()

    def refresh(self, field):
        for p in self.plans:
            for q, recv_idx in p.refresh_recv.items():
                self._move(field, q, self.plans[q].refresh_send[p.rank], p.rank, recv_idx)

    def pushback(self, colour):
        for p in self.plans:
            for (c, q), idx in p.pushback_send.items():
                if c != colour:
                    continue
                self._move("vel", p.rank, idx, q, self.plans[q].pushback_recv[(c, p.rank)])

    def allsum(self, values):
        return float(sum(values))

    def allmax(self, values):
        return float(max(values))

    def control(self, mode):
        """Device control step of every rank: the ranks' partials are
        gathered into one device buffer ([nranks][4], rank order) and every
        rank's control kernel reduces it (the all-gather of TorchGroup)."""
        import torch
        w = len(self.devices)
        if getattr(self, "_gat", None) is None or self._gat.numel() != 4 * w:
            self._gat = torch.zeros(4 * w, dtype=torch.float64, device="cuda")
        for r, dev in enumerate(self.devices):
            dev.rank_partials(mode, self._gat.data_ptr() + 32 * r)
        for dev in self.devices:
            torch.cuda.ExternalStream(dev.stream_handle()).synchronize()
        for dev in self.devices:
            dev.control_ranks(self._gat.data_ptr(), w, mode)
        for dev in self.devices:
            torch.cuda.ExternalStream(dev.stream_handle()).synchronize()


class TorchGroup:
    """One rank per process; point-to-point exchanges and reductions through
    torch.distributed.

    tensor_device "cpu" (gloo): host-staged buffers (pack -> D2H -> send ->
    H2D -> unpack).  tensor_device "cuda" (NCCL): device-resident exchange --
    the index lists are mapped to the solid's internal ids and uploaded once,
    send/receive buffers are persistent CUDA tensors, and pack kernel ->
    NCCL isend/irecv -> unpack kernel are all ordered on the solid's own
    stream (torch.cuda.ExternalStream), with no host synchronisation."""

    def __init__(self, plan, device, dist, tensor_device="cpu"):
        import torch
        self.torch = torch
        self.dist = dist
        self.plans = [plan]
        self.devices = [device]
        self.tdev = tensor_device
        self.on_device = str(tensor_device).startswith("cuda")
        if self.on_device:
            self._setup_device_lists()
            # a global collective first, so the grouped send/recv of the
            # first exchange is never the first collective of the group
            dist.barrier()

    # -- device-resident exchange -------------------------------------
    def _setup_device_lists(self):
        torch = self.torch
        p, dev = self.plans[0], self.devices[0]
        d = dev.d

        def entry(idx, width):
            ids = torch.from_numpy(dev.internal_ids(idx)).to(self.tdev)
            return ids, torch.empty((len(idx), width), dtype=torch.float64, device=self.tdev)

        self.dl = {}
        fields = getattr(dev, "EXCHANGED", ("vel", "T"))
        for field, width in ((f, dev.field_width(f)) for f in fields):
            self.dl[("refresh_send", field)] = {q: entry(i, width) for q, i in p.refresh_send.items()}
            self.dl[("refresh_recv", field)] = {q: entry(i, width) for q, i in p.refresh_recv.items()}
        self.dl["push_send"] = {k: entry(i, d) for k, i in p.pushback_send.items()}
        self.dl["push_recv"] = {k: entry(i, d) for k, i in p.pushback_recv.items()}
        self.stream = torch.cuda.ExternalStream(dev.stream_handle())

    def _exchange_device(self, field, sends, recvs):
        """sends / recvs: {peer: (internal ids, buffer)} (CUDA tensors)."""
        torch, dist, dev = self.torch, self.dist, self.devices[0]
        with torch.cuda.stream(self.stream):
            for q, (ids, buf) in sorted(sends.items()):
                dev.pack_device(field, len(ids), ids.data_ptr(), buf.data_ptr())
            # one NCCL group (ncclGroupStart/End): separate isend/irecv calls
            # would each block their pair's stream until matched, and two
            # ranks that both receive first would deadlock
            ops = [dist.P2POp(dist.irecv, buf, q) for q, (ids, buf) in sorted(recvs.items())]
            ops += [dist.P2POp(dist.isend, buf, q) for q, (ids, buf) in sorted(sends.items())]
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()      # NCCL: the stream waits, the host does not
            for q, (ids, buf) in sorted(recvs.items()):
                dev.unpack_device(field, len(ids), ids.data_ptr(), buf.data_ptr())

    # -- host-staged exchange -----------------------------------------
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
        if self.on_device:
            self._exchange_device(field, self.dl[("refresh_send", field)],
                                  self.dl[("refresh_recv", field)])
            return
        p, dev = self.plans[0], self.devices[0]
        width = dev.field_width(field)
        sends = {q: dev.pack(field, idx) for q, idx in p.refresh_send.items()}
        got = self._swap(sends, {q: len(i) for q, i in p.refresh_recv.items()}, width)
        for q, vals in got.items():
            dev.unpack(field, p.refresh_recv[q], vals)

    def pushback(self, colour):
        if self.on_device:
            self._exchange_device(
                "vel", {q: e for (c, q), e in self.dl["push_send"].items() if c == colour},
                {q: e for (c, q), e in self.dl["push_recv"].items() if c == colour})
            return
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

    def control(self, mode):
        """Device control step: this rank's partials (4 doubles) are
        all-gathered into [world][4] and the control kernel applies the
        stopping rule and next step on every rank from the same numbers.
        NCCL: all on the solid's stream, no host synchronisation.  gloo:
        host-staged."""
        torch, dist, dev = self.torch, self.dist, self.devices[0]
        w = dist.get_world_size()
        if self.on_device:
            if getattr(self, "_loc", None) is None:
                self._loc = torch.zeros(4, dtype=torch.float64, device=self.tdev)
                self._gat = torch.zeros(4 * w, dtype=torch.float64, device=self.tdev)
            with torch.cuda.stream(self.stream):
                dev.rank_partials(mode, self._loc.data_ptr())
                dist.all_gather_into_tensor(self._gat, self._loc, async_op=True).wait()
                dev.control_ranks(self._gat.data_ptr(), w, mode)
            return
        loc = torch.from_numpy(np.ascontiguousarray(dev.rank_partials_host(mode), dtype=np.float64))
        out = [torch.zeros(4, dtype=torch.float64) for _ in range(w)]
        dist.all_gather(out, loc)
        dev.control_ranks_host(np.concatenate([o.numpy() for o in out]), mode)


def stable_dt(h, sound, cfl, vmax2, amax2):
    """solids.py:187, evaluated like the device control kernel."""
    dt = h / (sound + math.sqrt(vmax2))
    amax = math.sqrt(amax2)
    if amax > 0.0:
        dt = min(dt, math.sqrt(h / amax))
    return cfl * dt


class _GraphedStep:
    """CUDA-graph capture of one rank's inner step for the device-controlled
    loops: the phases (kernels on the problem's stream), the pack / unpack
    kernels, the grouped NCCL send/recv of every halo exchange and the NCCL
    all-gather + control kernel, recorded once and replayed per step.  Every
    kernel reads dt, the ramp counter and the done flag from the device control
    block, so a replay is the same step the eager enqueue would issue, without
    the ~40 phase calls and ~35 exchange calls from Python per step.  Only for
    TorchGroup on the device (NCCL); a capture that fails -- a torch / NCCL
    build that cannot capture the exchange -- falls back to the eager enqueue.
    MTSPH_DECOMP_GRAPH=1 / 0 forces it on / off; unset, it is on for a single
    rank and off for several (the graph with point-to-point NCCL nodes has not
    run on more than one GPU yet)."""

    _graph = None          # None: not tried, False: unavailable
    graph_replays = 0      # steps issued by replay (their launches are not in dev.launches())
    graph_launches = 0     # library launches of one captured step
    issue_s = 0.0          # host seconds spent issuing steps in relax_device
    issue_steps = 0

    def _issue_step(self):
        import os
        g = self.group
        if self._graph is None:
            self._graph = False
            # default: on for a single rank (exercised on hardware), and for
            # several ranks only on request -- the graph with point-to-point
            # NCCL nodes has never run on more than one GPU in this repository
            want = os.environ.get("MTSPH_DECOMP_GRAPH")
            if want is None:
                want = "1" if getattr(self, "nranks", 1) == 1 else "0"
            if getattr(g, "on_device", False) and want != "0":
                torch = g.torch
                dev = self.devices[0]
                # first step eagerly: lazily created exchange / control buffers
                # and NCCL's own first-use setup must not happen inside a capture
                self._step_async()
                try:
                    graph = torch.cuda.CUDAGraph()
                    l0 = dev.launches()
                    with torch.cuda.graph(graph, stream=g.stream, capture_error_mode="thread_local"):
                        self._step_async()
                    self.graph_launches = dev.launches() - l0
                    self._graph = graph
                except Exception as e:  # noqa: BLE001 -- any capture failure means "no graph"
                    import warnings
                    warnings.warn(f"decomposed step: CUDA graph capture unavailable ({type(e).__name__}: {e}); "
                                  "enqueueing the phases eagerly")
                    torch.cuda.synchronize()
                return
        if self._graph:
            with g.torch.cuda.stream(g.stream):
                self._graph.replay()
            self.graph_replays += 1
        else:
            self._step_async()


class DecomposedSolid(_GraphedStep):
    """A necking-type solid split into x-slabs (tiled damping sweep)."""

    def __init__(self, lat, elastic, hardening, nranks, ranks=None, group="local",
                 dist=None, tensor_device="cpu", end_disp_per_outer=0.0, ramp_steps=1):
        ranks = list(range(nranks)) if ranks is None else list(ranks)
        # one process per GPU builds only its own plan (and its neighbours'
        # exchange lists); the in-process emulation builds all of them
        self.plans, self.grid, self.owner = make_plans(
            lat.pos, lat.h_axes, nranks, ranks=None if group in ("local", "local_device") else ranks)
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
        if group in ("local", "local_device"):
            self.group = LocalGroup(self.plans, [devices[r] for r in range(nranks)],
                                    device_buffers=group == "local_device")
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
        self.nranks = int(nranks)

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

    # -- device-controlled loop ------------------------------------------
    def _step_async(self):
        g = self.group
        for dev in self.devices:
            dev.phase_async("kick_drift")
        g.refresh("vel")
        for dev in self.devices:
            dev.phase_async("stress")
        g.refresh("T")
        for dev in self.devices:
            dev.phase_async("accel")
        g.refresh("vel")
        if self.nranks == 1 and os.environ.get("MTSPH_DECOMP_COLOURS", "0") != "1":
            # one rank, no ghosts: the single-domain persistent dataflow
            # sweep (one launch, same tasks in the same order per particle).
            # MTSPH_DECOMP_COLOURS=1 keeps the multi-rank sequence (a launch,
            # push-back and refresh per colour and pass) for measuring its
            # issue cost on one GPU.
            self.devices[0].phase_async("sweep_all")
        else:
            nc = self.ncolours
            for rev in (False, True):
                for q in range(nc):
                    c = nc - 1 - q if rev else q
                    for dev in self.devices:
                        dev.phase_async("sweep", c + 64 if rev else c)
                    g.pushback(c)
                    g.refresh("vel")
        for dev in self.devices:
            dev.phase_async("vmax")
        g.control(1)

    def relax_device(self, eta, cfl, criterion, dt_outer, max_inner=0, min_inner=1,
                     fixed_steps=None, check_every=8):
        """The inner loop with the control on the device of every rank: the
        phases and exchanges are enqueued without host synchronisation, the
        ranks' reductions are all-gathered on the device and each rank's
        control kernel takes the same decisions (stepping.py:158 rule); the
        host reads the control block once every `check_every` steps.
        Returns (n_inner, ek, cap_hit, min_dt) like relax()."""
        if fixed_steps is not None:
            criterion, max_inner, min_inner = -1.0, int(fixed_steps), int(fixed_steps)
        for dev in self.devices:
            dev.begin_loop(eta, cfl, criterion, dt_outer, max_inner, min_inner)
            dev.set_ramp(self.end_disp, self.ramp_steps, self.ramp_left)
            dev.phase_async("amax")
        self.group.control(0)
        while True:
            t_issue = time.perf_counter()
            for _ in range(max(int(check_every), 1)):
                self._issue_step()
            self.issue_s += time.perf_counter() - t_issue   # host time to issue the steps (no sync inside)
            self.issue_steps += max(int(check_every), 1)
            states = [dev.loop_state() for dev in self.devices]
            if all(done for done, _ in states):
                break
        self.ramp_left = self.devices[0].ramp_left()
        r = states[0][1]
        return int(r.n_inner), float(r.ek), bool(r.cap_hit), float(r.min_dt)

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


class DecomposedPorous(_GraphedStep):
    """A porous membrane (PorousProblem) split into x-slabs: the outer
    diffusion step and the inner relaxation as device phases separated by
    ghost exchanges, with the host-side control of DecomposedSolid.relax.

    Exchanges per outer step: (s, V) after each preparation, the mass-update
    record after the first flux, the flux-rate record, 1/m_mix and v after
    the velocity split.  Per inner step: v after the kick, T~ after the
    constitutive update, v after the divergence, and per sweep colour the
    push-back and refresh of v, as in the solid.  Host-staged exchanges
    (LocalGroup, or TorchGroup with tensor_device="cpu")."""

    def __init__(self, lat, model, contact_time, evaporation_rate, nranks, ranks=None,
                 group="local", dist=None, tensor_device="cpu"):
        from .device import DevicePorous
        self.nranks = int(nranks)
        ranks = list(range(nranks)) if ranks is None else list(ranks)
        self.plans, self.grid, self.owner = make_plans(
            lat.pos, lat.h_axes, nranks, ranks=None if group in ("local", "local_device") else ranks)
        devices = {}
        for r in ranks:
            p = self.plans[r]
            ids = p.local_ids
            devices[r] = DevicePorous(lat.pos[ids], lat.vol[ids], lat.constrained[ids],
                                      lat.contact[ids], lat.h_axes, model, contact_time,
                                      evaporation_rate, sweep="tiled", ghost=p.ghost,
                                      grid=self.grid, tile=p.tile_B)
        if group in ("local", "local_device"):
            self.group = LocalGroup(self.plans, [devices[r] for r in range(nranks)],
                                    device_buffers=group == "local_device")
        else:
            (r,) = ranks
            self.group = TorchGroup(self.plans[r], devices[r], dist, tensor_device)
        self.devices = self.group.devices
        self.h = float(np.min(lat.h_axes))
        self.sound = math.sqrt(model.bulk_modulus / model.density0)
        # the reference sums the free volumes in original order
        self.vol_movable = float(np.sum(lat.vol[~np.asarray(lat.constrained, bool)]))
        self.ncolours = max(dev.colours() for dev in self.devices)
        self.n_global = len(lat.vol)

    def advance_slow(self, dt_outer, t):
        """PorousProblem.advance_slow: returns the number of clamped particles."""
        g = self.group
        for dev in self.devices:
            dev.set_outer(dt_outer, t)
            dev.phase("prep_map")
        g.refresh("satvol")
        for dev in self.devices:
            dev.phase("flux_mass")
        g.refresh("rm")
        clamped = g.allsum([dev.phase("mass")[0] for dev in self.devices])
        for dev in self.devices:
            dev.phase("prep")
        g.refresh("satvol")
        for dev in self.devices:
            dev.phase("flux")
            dev.phase("post")
        g.refresh("rf")
        g.refresh("inv_mix")
        g.refresh("vel")
        for dev in self.devices:
            dev.phase("fluxrate")
        return int(round(clamped))

    def step(self, dt, eta):
        g = self.group
        for dev in self.devices:
            dev.set_step(dt, eta)
            dev.phase("kick")
        g.refresh("vel")
        for dev in self.devices:
            dev.phase("stress")
        g.refresh("T")
        parts = [dev.phase("accel") for dev in self.devices]
        ek = 0.5 * g.allsum([p[0] for p in parts]) / self.vol_movable
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
        vmax2 = g.allmax([dev.phase("post_step")[0] for dev in self.devices])
        return ek, vmax2, amax2

    def initial_dt(self, cfl):
        vals = [dev.phase("amax") for dev in self.devices]
        return stable_dt(self.h, self.sound, cfl, self.group.allmax([v[0] for v in vals]),
                         self.group.allmax([v[1] for v in vals]))

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
                if ek <= criterion and n >= min_inner:
                    return n, ek, False, min_dt
                if n >= cap:
                    return n, ek, True, min_dt
            dt = stable_dt(self.h, self.sound, cfl, vmax2, amax2)

    # -- device-controlled inner loop (as DecomposedSolid.relax_device) -----
    def _step_async(self):
        g = self.group
        for dev in self.devices:
            dev.phase_async("kick")
        g.refresh("vel")
        for dev in self.devices:
            dev.phase_async("stress")
        g.refresh("T")
        for dev in self.devices:
            dev.phase_async("accel")
        g.refresh("vel")
        nc = self.ncolours
        for rev in (False, True):
            for q in range(nc):
                c = nc - 1 - q if rev else q
                for dev in self.devices:
                    dev.phase_async("sweep", c + 64 if rev else c)
                g.pushback(c)
                g.refresh("vel")
        for dev in self.devices:
            dev.phase_async("post_step")
        g.control(1)

    def relax_device(self, eta, cfl, criterion, dt_outer, max_inner=0, min_inner=1,
                     fixed_steps=None, check_every=8):
        """Inner loop with phases enqueued without host synchronisation and
        the stopping rule applied on every rank's device from all-gathered
        partials; E_k normalised by the whole problem's free volume."""
        if fixed_steps is not None:
            criterion, max_inner, min_inner = -1.0, int(fixed_steps), int(fixed_steps)
        for dev in self.devices:
            dev.begin_loop(eta, cfl, criterion, dt_outer, max_inner, min_inner,
                           vol_movable=self.vol_movable)
            dev.phase_async("amax")
        self.group.control(0)
        while True:
            t_issue = time.perf_counter()
            for _ in range(max(int(check_every), 1)):
                self._issue_step()
            self.issue_s += time.perf_counter() - t_issue   # host time to issue the steps (no sync inside)
            self.issue_steps += max(int(check_every), 1)
            states = [dev.loop_state() for dev in self.devices]
            if all(done for done, _ in states):
                break
        r = states[0][1]
        return int(r.n_inner), float(r.ek), bool(r.cap_hit), float(r.min_dt)

    def gather(self, field):
        """Owned values of `field` in global particle order (LocalGroup only)."""
        sample = self.devices[0].get(field)
        out = np.zeros((self.n_global,) + sample.shape[1:])
        for p, dev in zip(self.plans, self.devices):
            vals = dev.get(field)
            own = ~p.ghost
            out[p.local_ids[own]] = vals[own]
        return out
