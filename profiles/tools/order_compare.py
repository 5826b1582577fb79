"""The reference's desk-resolution necking acceptance run (dp = PH/25, 1000
outer steps) in the reference damping order (`serial`, parity mode) and in
the B200 tiled order: how far the tiled order's observables move from the
reference order's over a whole run with plastic flow and necking.

    python profiles/tools/order_compare.py > profiles/order_compare_r01.json
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

from paper_2309_04010_b200.config import resolve  # noqa: E402
from paper_2309_04010_b200.scenarios import build  # noqa: E402
from paper_2309_04010_b200.stepping import run_outer_inner  # noqa: E402

p = resolve({"scenario": "necking_2d", "dp": 12.826e-3 / 25, "n_outer": 1000}).params
runs = {}
for sweep in ("serial", "tiled"):
    problem, policy = build(p, sweep=sweep)
    t0 = time.perf_counter()
    obs, counters = run_outer_inner(problem, policy)
    runs[sweep] = {"obs": obs, "n_inner": int(counters.n_inner), "s": time.perf_counter() - t0,
                   "u": problem.state.pos - problem.state.ref_pos}
a, b = runs["serial"], runs["tiled"]
fa, fb = a["obs"].reaction_force, b["obs"].reaction_force
peak = float(np.max(fa))
iy = {k: int(np.argmax(r["obs"].extras["mid_alpha_min"] > 0)) for k, r in runs.items()}
out = {
    "workload": "necking_2d desk (dp = PH/25, 2600 particles), 1000 outer steps",
    "wall_s": {k: round(r["s"], 1) for k, r in runs.items()},
    "inner_steps": {k: r["n_inner"] for k, r in runs.items()},
    "peak_force": {"serial": peak, "tiled": float(np.max(fb))},
    "force_curve_max_diff_over_peak": float(np.max(np.abs(fa - fb)) / peak),
    "neck_disp_final": {"serial": float(a["obs"].neck_disp[-1]), "tiled": float(b["obs"].neck_disp[-1])},
    "first_midspan_yield_step": iy,
    "displacement_rel_l2": float(np.linalg.norm(a["u"] - b["u"]) / np.linalg.norm(a["u"])),
}
print(json.dumps(out))
