"""Tuning sweep (GPU): lanes per particle of the row-parallel gathers, one
solid, both precisions.  Prints per-class device ms per step (CUDA events
in the step graph).

    python profiles/tools/tune_lanes.py [--dp 0.02] [--steps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bar_3d")
    ap.add_argument("--dp", type=float, default=0.0)
    ap.add_argument("--sweep", default="tiled")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--lanes32", default="4,8,16,2")
    args = ap.parse_args()
    params = bench.workload_params(args)
    dev, lat, _, _ = bench.build_solid(params, args.sweep)
    eta, cfl = params["eta"], params["cfl"]

    def timed(tag):
        dev.run_steps(args.steps, eta, cfl)
        t = dev.run_steps(args.steps, eta, cfl)
        out = {k: round(v / args.steps, 3) for k, v in t.items() if k.endswith("_ms")}
        print(tag, json.dumps(out), flush=True)

    timed("fp64 lanes=4")
    for g in args.lanes32.split(","):
        os.environ["MTSPH_GATHER_LANES32"] = g
        dev.set_precision(32)
        timed(f"fp32 lanes={g}")
        dev.set_precision(64)


if __name__ == "__main__":
    main()
