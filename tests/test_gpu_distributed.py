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
