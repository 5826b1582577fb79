"""Mirror symmetry of the damping orders on the reference's 3D acceptance
smoke cases (test_acceptance.py:441-540): the necking_3d bar (transverse
mirror of the displacement) and the fsi_3d film (two-plane mirror of the
deflection), each run through the drop-in driver in the serial (reference),
coloured and tiled orders.  Prints one JSON line per run.

    python profiles/tools/symmetry_probe.py > profiles/parity_r02/symmetry_3d.jsonl
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import test_gpu_acceptance_3d as A  # noqa: E402

for name, raw, measure in (("necking_3d", A.NECK3D, A._neck_symmetry),
                           ("fsi_3d", A.FSI3D, A._fsi_symmetry)):
    for sweep in ("serial", "coloured", "tiled"):
        t0 = time.perf_counter()
        run = A._run(raw, sweep)
        obs = run["obs"]
        print(json.dumps({"case": name, "order": sweep, "mirror_asymmetry_rel": measure(run),
                          "n_inner_total": int(np.sum(obs.n_inner)),
                          "cap_hits": len(run["counters"].cap_hits),
                          "amplitude_last": float(obs.amplitude[-1]),
                          "wall_s": round(time.perf_counter() - t0, 1)}), flush=True)
