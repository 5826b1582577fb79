"""Damping-order parity under the BASELINE loading (profiles/tools).

Runs a necking-type scenario twice through the drop-in driver protocol
(scenarios.build + the device inner loop), once in the reference's damping
order (serial) and once in a parallel order, with the BASELINE loading
(right end pulled at 1e-3 length units per unit time, outer dt 0.01,
inner loop capped at the reference's 10 ceil(dt_outer/dt)), then relaxes
both to E_k <= criterion and prints the relative L2 differences of the
displacement, F, C_p^-1 and alpha fields at every checkpoint.

    python profiles/tools/loading_parity.py --scenario bar_2d --checkpoints 250,500,1000
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scenario", default="bar_2d")
    ap.add_argument("--length", type=float, default=0.0)
    ap.add_argument("--width", type=float, default=0.0)
    ap.add_argument("--breadth", type=float, default=0.0)
    ap.add_argument("--pre", type=float, default=0.0,
                    help="first apply this fraction of the yield end displacement "
                         "(sigma0/E x length) by a slow ramp and relax")
    ap.add_argument("--pre-ramp", type=int, default=4000)
    ap.add_argument("--checkpoints", default="250,500,1000")
    ap.add_argument("--orders", default="tiled")
    ap.add_argument("--final-criterion", type=float, default=1e-8)
    ap.add_argument("--final-max", type=int, default=400000)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    from paper_2309_04010_b200 import scenarios
    from paper_2309_04010_b200.config import resolve
    raw = {"scenario": args.scenario}
    for k in ("length", "width", "breadth"):
        if getattr(args, k):
            raw[k] = getattr(args, k)
    p = resolve(raw).params
    cps = [int(c) for c in args.checkpoints.split(",")]
    orders = ["serial"] + args.orders.split(",")
    probs = {}
    for o in orders:
        probs[o] = scenarios.build(p, sweep=o)
    n = probs["serial"][0].lattice.n
    pol = probs["serial"][1]
    rate = p["stretch_per_end"] / p["n_outer"] / pol.dt_outer
    print(json.dumps({"scenario": args.scenario, "particles": n, "dt_outer": pol.dt_outer,
                      "pull_rate": rate, "eta": pol.eta, "criterion": pol.energy_criterion}),
          flush=True)
    if args.pre > 0:
        e_mod = 9 * p["bulk_modulus"] * p["shear_modulus"] / (3 * p["bulk_modulus"] + p["shear_modulus"])
        disp = args.pre * p["initial_flow_stress"] / e_mod * p["length"]
        for o in orders:
            prob, _ = probs[o]
            t0 = time.perf_counter()
            prob.dev.set_ramp(disp, args.pre_ramp, args.pre_ramp)
            r = prob.dev.relax(pol.eta, pol.cfl, args.final_criterion, pol.dt_outer,
                               max_inner=args.final_max, min_inner=1)
            print(f"  {o}: pre-stretch {disp:.4g} in {int(r.n_inner)} steps cap_hit {int(r.cap_hit)} "
                  f"({time.perf_counter() - t0:.1f} s)", flush=True)
    done = {o: 0 for o in orders}
    inner = {o: 0 for o in orders}
    caps = {o: 0 for o in orders}
    rows = []
    for cp in cps:
        for o in orders:
            prob, _ = probs[o]
            t0 = time.perf_counter()
            while done[o] < cp:
                done[o] += 1
                prob.advance_slow(done[o], pol.dt_outer, done[o] * pol.dt_outer)
                nin, rep, capped, _ = prob.relax_inner(pol)
                inner[o] += nin
                caps[o] += int(capped)
            # snapshot, relax a copy-free way: relax to the criterion (the
            # loading continues from the relaxed state afterwards in both)
            r = prob.dev.relax(pol.eta, pol.cfl, args.final_criterion, pol.dt_outer,
                               max_inner=args.final_max, min_inner=1)
            inner[o] += int(r.n_inner)
            print(f"  {o}: outer {done[o]}, final relax {int(r.n_inner)} steps cap_hit "
                  f"{int(r.cap_hit)} ek {r.ek:.3e}  ({time.perf_counter() - t0:.1f} s)", flush=True)
        ref = probs["serial"][0]
        d_ref = ref.dev
        u_ref = d_ref.get("pos") - ref.lattice.pos
        f_ref = d_ref.get("F")
        c_ref = d_ref.get("cp_inv")
        a_ref = d_ref.get("alpha")
        eye = np.eye(u_ref.shape[1])
        from oracle import oracle as O
        from paper_2309_04010_b200.scenarios import _necking_materials
        _, hard = _necking_materials(p)
        law, hp = hard.device_params()
        matp = O.material_vector(p["shear_modulus"], p["bulk_modulus"], *hp, law=law)

        def stress(dv):   # Kirchhoff stress of the current state (trial = converged)
            return O.return_map(dv.get("F"), dv.get("cp_inv"), dv.get("alpha"), matp)[0]
        t_ref = stress(d_ref)
        row = {"outer": cp, "max_alpha": float(a_ref.max()),
               "plastic_frac": float(np.mean(a_ref > 0)), "inner": dict(inner), "caps": dict(caps)}
        for o in orders[1:]:
            dv = probs[o][0].dev
            u = dv.get("pos") - ref.lattice.pos
            row[o] = {"u": rel(u, u_ref), "F": rel(dv.get("F") - eye, f_ref - eye),
                      "tau": rel(stress(dv), t_ref),
                      "cp_inv": rel(dv.get("cp_inv") - eye, c_ref - eye) if a_ref.max() > 0 else 0.0,
                      "alpha": rel(dv.get("alpha"), a_ref) if a_ref.max() > 0 else 0.0}
        rows.append(row)
        print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
