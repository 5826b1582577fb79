"""Application run at benchmark scale (GPU): the reference driver protocol
(stepping.run_outer_inner) on BASELINE configs[2] -- the 10 M-particle 3D
power-law bar, left end clamped, right end pulled at the BASELINE rate, outer
dt 0.01 -- with every inner loop on the device (graph chunks, stopping rule
in the control kernel).  Prints one JSON line: inner steps per outer step,
wall time, observables.

    python profiles/tools/app_run.py [--n-outer 3] [--sweep tiled] [--fp32]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-outer", type=int, default=3)
    ap.add_argument("--sweep", default="tiled")
    ap.add_argument("--fp32", action="store_true")
    ap.add_argument("--scenario", default="bar_3d", help="bar_3d (configs[2]) or block_3d (configs[4])")
    ap.add_argument("--length", type=float, default=0.0)
    ap.add_argument("--max-inner", type=int, default=0,
                    help="inner cap (0: the reference's 10 ceil(dt_outer/dt))")
    ap.add_argument("--membrane", action="store_true",
                    help="the BASELINE configs[3] plate (membrane_3d, 17.1 M particles)")
    args = ap.parse_args()
    if args.membrane:
        return membrane(args)
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.stepping import run_outer_inner
    base = resolve({"scenario": args.scenario}).params
    dt_outer = base["t_total"] / base["n_outer"]
    raw = {"scenario": args.scenario, "n_outer": args.n_outer, "t_total": args.n_outer * dt_outer,
           "stretch_per_end": base["stretch_per_end"] * args.n_outer / base["n_outer"],
           "damping_sweep": args.sweep, "max_inner": args.max_inner}
    if args.length:
        raw["length"] = args.length
    p = resolve(raw).params
    t0 = time.perf_counter()
    problem, policy = scenarios.build(p, sweep=args.sweep)
    setup = time.perf_counter() - t0
    if args.fp32:
        problem.dev.set_precision(32)
    t0 = time.perf_counter()
    obs, counters = run_outer_inner(problem, policy)
    wall = time.perf_counter() - t0
    n = problem.lattice.n
    print(json.dumps({
        "workload": f"{args.scenario} (BASELINE configs[{2 if args.scenario == 'bar_3d' else 4}]), "
                    f"{n} particles, {args.sweep} sweep, "
                    f"{'fp32 variant' if args.fp32 else 'fp64'}",
        "dt_outer": policy.dt_outer, "energy_criterion": policy.energy_criterion,
        "n_outer": counters.n_outer, "n_inner": [int(x) for x in obs.n_inner],
        "ek_ratio": [float(x) for x in obs.ek_ratio], "max_inner": p["max_inner"],
        "cap_hits": counters.cap_hits, "setup_s": setup, "wall_s": wall,
        "inner_steps_per_s": counters.n_inner / wall,
        "particle_steps_per_s": n * counters.n_inner / wall,
        "reaction_force": [float(x) for x in obs.reaction_force],
        "min_dt_inner": counters.min_dt_inner}))


def membrane(args):
    import numpy as np
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.stepping import run_outer_inner
    base = resolve({"scenario": "membrane_3d"}).params
    dt_outer = base["t_total"] / base["n_outer"]
    p = resolve({"scenario": "membrane_3d", "n_outer": args.n_outer,
                 "t_total": args.n_outer * dt_outer, "damping_sweep": "tiled",
                 "max_inner": args.max_inner or 300}).params
    t0 = time.perf_counter()
    problem, policy = scenarios.build(p, sweep="tiled")
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    obs, counters = run_outer_inner(problem, policy)
    wall = time.perf_counter() - t0
    n = problem.lattice.n
    print(json.dumps({
        "workload": f"membrane_3d plate (BASELINE configs[3]) 40 x 40 x 1, {n} particles, tiled",
        "dt_outer": policy.dt_outer, "n_outer": counters.n_outer,
        "n_inner": [int(x) for x in obs.n_inner], "cap_hits": counters.cap_hits,
        "clamp_events": counters.clamp_events, "setup_s": setup, "wall_s": wall,
        "particle_steps_per_s": n * counters.n_inner / wall,
        "fluid_mass_total": [float(x) for x in obs.extras.get("fluid_mass_total", [])],
        "amplitude": [float(x) for x in obs.amplitude]}))


if __name__ == "__main__":
    main()
