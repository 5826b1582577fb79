"""Profiling driver (run under ncu): build the bench workload, run one fp64
inner step and one fp32 step through the step graph.  Not a bench: numbers
printed under a profiler are never reported.

    ncu --set full --clock-control none --import-source on \
        -k regex:'k_sweep_flow|k32_|k_solid_' -c 16 -o gpurun_out/step \
        python profiles/tools/prof_step.py [--dp 0.02] [--workload bar_3d]
"""
import argparse
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
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--precisions", default="64,32")
    ap.add_argument("--length", type=float, default=0.0)
    args = ap.parse_args()
    params = dict(bench.workload_params(args))
    if args.length:
        params["length"] = args.length
    dev, lat, _, _ = bench.build_solid(params, args.sweep)
    for bits in [int(b) for b in args.precisions.split(",")]:
        dev.set_precision(bits)
        dev.run_steps(args.steps, params["eta"], params["cfl"])
    print("profiled", lat.n, "particles")


if __name__ == "__main__":
    main()
