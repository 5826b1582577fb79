"""Per-step cost of the reference-order (serial) damping sweep at the
reference's acceptance sizes: the shared-memory kernel, the global-memory
kernel (MTSPH_SERIAL_SMEM=0), the tiled sweep and no sweep, timed through
the device inner loop (fixed step counts, wall clock around relax()).

    python profiles/tools/serial_probe.py > profiles/serial_probe_r01.jsonl
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from paper_2309_04010_b200.config import resolve  # noqa: E402
from paper_2309_04010_b200.scenarios import build  # noqa: E402

CASES = {"necking_2d desk (dp = PH/25)": {"scenario": "necking_2d", "dp": 12.826e-3 / 25,
                                          "n_outer": 1000},
         "fsi_2d paper scale": {"scenario": "fsi_2d"}}
STEPS = 400

for name, raw in CASES.items():
    p = resolve(raw).params
    for label, sweep, smem in (("serial, shared memory", "serial", "1"),
                               ("serial, global memory", "serial", "0"),
                               ("tiled", "tiled", "1"), ("none", "none", "1")):
        os.environ["MTSPH_SERIAL_SMEM"] = smem
        problem, policy = build(p, sweep=sweep)
        dev = problem.dev
        if hasattr(dev, "set_ramp"):
            dev.set_ramp(problem.end_disp_per_outer, problem.ramp_steps, problem.ramp_steps)
        else:
            dev.advance_slow(policy.dt_outer, policy.dt_outer)
        kw = dict(eta=policy.eta, cfl=policy.cfl, criterion=-1.0, dt_outer=policy.dt_outer)
        dev.relax(max_inner=20, min_inner=20, **kw)
        t0 = time.perf_counter()
        dev.relax(max_inner=STEPS, min_inner=STEPS, **kw)
        ms = (time.perf_counter() - t0) * 1e3 / STEPS
        sz = dev.sizes()
        print(json.dumps({"case": name, "sweep": label, "particles": int(problem.state.n),
                          "pairs": sz["npairs"] if isinstance(sz, dict) else int(sz[1]),
                          "levels": sz["phases"] if isinstance(sz, dict) else int(sz[3]),
                          "ms_per_inner_step": round(ms, 4)}), flush=True)
