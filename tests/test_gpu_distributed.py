"""GPU: the slab-decomposed inner step reproduces the single-domain tiled
pipeline.  All ranks run in one process on one GPU (LocalGroup) -- no
kernel waits on another rank.  Exchanges are host-staged copies, or the
device-resident path of the NCCL group (internal-id lists and buffers on
the device, pack / unpack kernels on each solid's stream) with a device copy
in place of the NCCL send/recv."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(length=0.8):
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.scenarios import _necking_materials
    p = resolve({"scenario": "block_3d", "length": length, "width": 0.12, "breadth": 0.12}).params
    lat = lattices.build_lattice(p)
    el, hard = _necking_materials(p)
    return p, lat, el, hard


@pytest.mark.parametrize("group", ["local", "local_device"])
def test_decomposed_matches_single_domain_tiled(group):
    from paper_2309_04010_b200.device import DeviceSolid
    from paper_2309_04010_b200.distributed import DecomposedSolid
    p, lat, el, hard = _setup()
    law, hp = hard.device_params()
    steps, eta, cfl = 25, p["eta"], p["cfl"]
    end_disp = 0.02 * p["length"]
    # production single-domain path: stable_dt + relax_step over the C ABI
    ref = DeviceSolid(lat.pos, lat.vol, el.density0, lat.constrained, lat.side, lat.mid_mask,
                      lat.h_axes, el.shear_modulus, el.bulk_modulus, plastic=True,
                      hardening_law=law, hard=hp, sweep="tiled")
    ref.set_ramp(end_disp, 10, 10)
    for _ in range(steps):
        ref.relax_step(ref.stable_dt(cfl), eta)
    want = {f: ref.get(f) for f in ("pos", "vel", "F", "alpha")}
    assert np.max(want["alpha"]) > 0
    for nranks in (1, 2, 3):
        dec = DecomposedSolid(lat, el, hard, nranks, group=group, end_disp_per_outer=end_disp,
                              ramp_steps=10)
        assert sum((~pl.ghost).sum() for pl in dec.plans) == len(lat.vol)
        dec.advance_slow()
        dec.relax(eta, cfl, 0.0, 1.0, fixed_steps=steps)
        for f, w in want.items():
            got = dec.gather(f)
            scale = max(np.max(np.abs(w)), 1e-300)
            err = np.max(np.abs(got - w)) / scale
            assert err <= 1e-13, (nranks, f, err)


@pytest.mark.parametrize("group", ["local", "local_device"])
def test_device_controlled_loop_matches_single_domain(group):
    """relax_device: phases enqueued without host synchronisation, rank
    partials gathered on the device, the control kernel of every rank takes
    the step decisions -- same trajectory as the single domain (fixed steps)
    and the same stopping step as the host-controlled decomposed loop."""
    from paper_2309_04010_b200.device import DeviceSolid
    from paper_2309_04010_b200.distributed import DecomposedSolid
    p, lat, el, hard = _setup()
    law, hp = hard.device_params()
    steps, eta, cfl = 25, p["eta"], p["cfl"]
    end_disp = 0.02 * p["length"]
    ref = DeviceSolid(lat.pos, lat.vol, el.density0, lat.constrained, lat.side, lat.mid_mask,
                      lat.h_axes, el.shear_modulus, el.bulk_modulus, plastic=True,
                      hardening_law=law, hard=hp, sweep="tiled")
    ref.set_ramp(end_disp, 10, 10)
    for _ in range(steps):
        ref.relax_step(ref.stable_dt(cfl), eta)
    want = {f: ref.get(f) for f in ("pos", "vel", "F", "alpha")}
    for nranks in (1, 2, 3):
        dec = DecomposedSolid(lat, el, hard, nranks, group=group, end_disp_per_outer=end_disp,
                              ramp_steps=10)
        dec.advance_slow()
        n, ek, cap, _ = dec.relax_device(eta, cfl, 0.0, 1.0, fixed_steps=steps, check_every=4)
        assert n == steps and dec.ramp_left == 0
        for f, w in want.items():
            got = dec.gather(f)
            scale = max(np.max(np.abs(w)), 1e-300)
            err = np.max(np.abs(got - w)) / scale
            assert err <= 1e-13, (nranks, f, err)
    # stopping rule: device-controlled and host-controlled loops agree
    crit = None
    for mode in ("host", "device"):
        dec = DecomposedSolid(lat, el, hard, 2, group=group, end_disp_per_outer=end_disp,
                              ramp_steps=10)
        dec.advance_slow()
        if crit is None:
            # a criterion the loop reaches after a few dozen steps
            n0, ek0, _, _ = dec.relax(eta, cfl, 0.0, 1.0, fixed_steps=40)
            # just above the step-40 energy, so that neither loop's rounding
            # (different summation orders) sits on the edge of the criterion
            crit = ek0 * (1.0 + 1e-6)
            continue
        n, ek, cap, _ = dec.relax_device(eta, cfl, crit, 1.0, max_inner=400)
        assert not cap and n <= 40 + 1
    dec_h = DecomposedSolid(lat, el, hard, 2, group=group, end_disp_per_outer=end_disp,
                            ramp_steps=10)
    dec_h.advance_slow()
    nh, ekh, caph, _ = dec_h.relax(eta, cfl, crit, 1.0, max_inner=400)
    assert n == nh and not caph
    assert abs(ek - ekh) <= 1e-12 * abs(ekh)


def test_nccl_group_single_rank_device_loop():
    """TorchGroup over a real NCCL communicator (world size 1 on this GPU):
    device-resident exchanges (none for one rank) and the NCCL all-gather of
    the control partials on the solid's stream, against the single domain."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2309_04010_b200.device import DeviceSolid
    from paper_2309_04010_b200.distributed import DecomposedSolid
    p, lat, el, hard = _setup()
    law, hp = hard.device_params()
    steps, eta, cfl = 20, p["eta"], p["cfl"]
    end_disp = 0.02 * p["length"]
    ref = DeviceSolid(lat.pos, lat.vol, el.density0, lat.constrained, lat.side, lat.mid_mask,
                      lat.h_axes, el.shear_modulus, el.bulk_modulus, plastic=True,
                      hardening_law=law, hard=hp, sweep="tiled")
    ref.set_ramp(end_disp, 10, 10)
    for _ in range(steps):
        ref.relax_step(ref.stable_dt(cfl), eta)
    want = {f: ref.get(f) for f in ("pos", "vel", "F")}
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        dec = DecomposedSolid(lat, el, hard, 1, ranks=[0], group="torch", dist=dist,
                              tensor_device="cuda", end_disp_per_outer=end_disp, ramp_steps=10)
        dec.advance_slow()
        n, ek, cap, _ = dec.relax_device(eta, cfl, 0.0, 1.0, fixed_steps=steps, check_every=5)
        assert n == steps
        # the step was captured in a CUDA graph (phases + NCCL all-gather +
        # control kernel) after its first eager issue, and replayed
        assert dec._graph, "graph capture of the decomposed step failed"
        assert dec.graph_replays == steps - 1 and dec.graph_launches > 0
        dev = dec.devices[0]
        for f, w in want.items():
            got = dev.get(f)
            scale = max(np.max(np.abs(w)), 1e-300)
            assert np.max(np.abs(got - w)) <= 1e-13 * scale, f
    finally:
        dist.destroy_process_group()


POROUS_CASES = {
    "membrane_2d": {"scenario": "membrane_2d"},
    "film_3d": {"scenario": "fsi_3d", "length": 4e-3, "breadth": 1e-3},
}


@pytest.mark.parametrize("group", ["local", "local_device"])
@pytest.mark.parametrize("case", sorted(POROUS_CASES))
@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_decomposed_porous_matches_single_domain(nranks, case, group):
    """The porous membrane (BASELINE configs[1] strip, wetted top face; the
    reference's 3D film, wetted centre) split into x-slabs: outer diffusion steps and inner relaxation as device phases
    with host-staged ghost exchanges reproduce the single domain (same tiled
    schedule) to 1e-12."""
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.device import DevicePorous
    from paper_2309_04010_b200.distributed import DecomposedPorous
    from paper_2309_04010_b200.scenarios import _membrane
    p = resolve(POROUS_CASES[case]).params
    lat = lattices.build_lattice(p)
    model = _membrane(p)
    dt_outer = p["t_total"] / max(p["n_outer"], 1)
    if case == "film_3d":
        dt_outer = 1.0
    ref = DevicePorous(lat.pos, lat.vol, lat.constrained, lat.contact, lat.h_axes, model,
                       p["contact_time"], p["evaporation_rate"], sweep="tiled")
    dec = DecomposedPorous(lat, model, p["contact_time"], p["evaporation_rate"], nranks,
                           group=group)
    assert sum((~pl.ghost).sum() for pl in dec.plans) == lat.n
    eta, cfl = p["eta"], p["cfl"]
    for step in (1, 2):
        t = step * dt_outer
        c_ref = ref.advance_slow(dt_outer, t)
        c_dec = dec.advance_slow(dt_outer, t)
        assert c_ref == c_dec
        dt = ref.stable_dt(cfl)
        assert abs(dec.initial_dt(cfl) - dt) <= 1e-12 * dt
        for _ in range(12):
            ek_ref = ref.relax_step(dt, eta)
            ek, _, _ = dec.step(dt, eta)
        assert abs(ek - ek_ref) <= 1e-10 * max(abs(ek_ref), 1e-300)
    for field in ("fluid_mass", "saturation", "pos", "F"):
        want = ref.get(field)
        got = dec.gather(field)
        scale = max(float(np.max(np.abs(want))), 1e-300)
        err = float(np.max(np.abs(got - want))) / scale
        assert err <= 1e-12, (nranks, field, err)
    assert float(np.max(ref.get("fluid_mass"))) > 0


@pytest.mark.parametrize("group", ["local", "local_device"])
def test_decomposed_porous_device_loop(group):
    """Device-controlled porous inner loop (phases enqueued, rank partials
    gathered on the device, per-rank control kernel) against the single
    domain's device loop: same steps, same state to 1e-12."""
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.device import DevicePorous
    from paper_2309_04010_b200.distributed import DecomposedPorous
    from paper_2309_04010_b200.scenarios import _membrane
    p = resolve({"scenario": "membrane_2d"}).params
    lat = lattices.build_lattice(p)
    model = _membrane(p)
    dt_outer = p["t_total"] / p["n_outer"]
    ref = DevicePorous(lat.pos, lat.vol, lat.constrained, lat.contact, lat.h_axes, model,
                       p["contact_time"], p["evaporation_rate"], sweep="tiled")
    dec = DecomposedPorous(lat, model, p["contact_time"], p["evaporation_rate"], 3, group=group)
    for step in (1, 2):
        t = step * dt_outer
        ref.advance_slow(dt_outer, t)
        dec.advance_slow(dt_outer, t)
        r = ref.relax(p["eta"], p["cfl"], -1.0, dt_outer, max_inner=15, min_inner=15)
        n, ek, cap, _ = dec.relax_device(p["eta"], p["cfl"], -1.0, dt_outer, fixed_steps=15,
                                         check_every=4)
        assert n == r.n_inner == 15
        assert abs(ek - r.ek) <= 1e-10 * max(abs(r.ek), 1e-300)
    for field in ("fluid_mass", "pos", "F"):
        want = ref.get(field)
        got = dec.gather(field)
        scale = max(float(np.max(np.abs(want))), 1e-300)
        assert float(np.max(np.abs(got - want))) / scale <= 1e-12, field


@pytest.mark.parametrize("group", ["local", "local_device"])
def test_error_on_one_rank_fails_every_rank(group):
    """An element inversion on rank 1 only: rank 1 raises
    ElementInversionError with the particle's id, and rank 0 -- which has no
    error of its own -- raises SimulationError instead of returning a normal
    result (its host would otherwise go on to the next outer step's exchanges
    alone and hang).  The flag travels in the all-gathered control partials."""
    from paper_2309_04010_b200.distributed import DecomposedSolid
    from paper_2309_04010_b200.errors import ElementInversionError, SimulationError
    p, lat, el, hard = _setup()
    dec = DecomposedSolid(lat, el, hard, 2, group=group)
    plan = dec.plans[1]
    own = np.flatnonzero(~plan.ghost & ~lat.constrained[plan.local_ids])
    victim = int(own[len(own) // 2])
    dev1 = dec.devices[1]
    F = dev1.get("F")
    F[victim] = np.diag([-1.0, 1.0, 1.0])
    dev1.set("F", F)
    with pytest.raises((ElementInversionError, SimulationError)):
        dec.relax_device(p["eta"], p["cfl"], 0.0, 1.0, fixed_steps=4, check_every=2)
    with pytest.raises(ElementInversionError) as e1:
        dec.devices[1].loop_state()
    assert int(plan.local_ids[victim]) in e1.value.particle_ids or victim in e1.value.particle_ids
    with pytest.raises(SimulationError, match="another rank"):
        dec.devices[0].loop_state()
