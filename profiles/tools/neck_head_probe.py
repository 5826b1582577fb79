import dataclasses, sys, json
sys.path.insert(0, ".")
import numpy as np
from paper_2309_04010_b200.config import resolve
from paper_2309_04010_b200.scenarios import build
from paper_2309_04010_b200.stepping import run_outer_inner
for sweep in ("serial", "tiled"):
    p = resolve({"scenario": "necking_2d", "dp": 12.826e-3 / 25, "n_outer": 1000}).params
    problem, policy = build(p, sweep=sweep)
    rows = []
    obs, c = run_outer_inner(problem, dataclasses.replace(policy, n_outer=14),
                             observers=[lambda s, t, smp: rows.append(smp)])
    print(sweep, "n_inner", obs.n_inner.tolist())
    for i, r in enumerate(rows):
        print(i, r)
