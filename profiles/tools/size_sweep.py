"""Throughput against problem size on one GPU (BASELINE configs[4]: the
jittered elastic-plastic block at 4M / 8M / 16M / 32M particles; the block
is lengthened along x at dp = 0.02).  fp64 and the fp32 variant, CUDA-event
timing of the step graph as in bench.py.  One JSON line per size.

    python profiles/tools/size_sweep.py [--lengths 8,16,32,64] [--steps 10]
"""
import argparse
import gc
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="8,16,32,64")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    from paper_2309_04010_b200.config import resolve
    for length in [float(x) for x in args.lengths.split(",")]:
        params = resolve({"scenario": "block_3d", "length": length, "damping_sweep": "tiled"}).params
        t0 = time.perf_counter()
        dev, lat, _, setup = bench.build_solid(params, "tiled")
        out = {"workload": f"block_3d {length:g} x 2 x 2, dp 0.02, jitter 0.05 (BASELINE configs[4])",
               "particles": int(lat.n), "setup_s": round(setup, 1)}
        sz = dev.sizes()
        out["neighbours_per_particle"] = sz["nnz"] / lat.n
        for bits in (64, 32):
            dev.set_precision(bits)
            dev.run_steps(args.steps, params["eta"], params["cfl"])
            t = dev.run_steps(args.steps, params["eta"], params["cfl"])
            ms = t["total_ms"] / args.steps
            out[f"fp{bits}"] = {"ms_per_step": ms, "particle_steps_per_s": lat.n / (ms / 1e3),
                                 "kernels_ms": {k[:-3]: round(v / args.steps, 3) for k, v in t.items()
                                                if k.endswith("_ms") and k != "total_ms"},
                                 "finite": dev.measure()["finite"]}
        print(json.dumps(out), flush=True)
        del dev, lat
        gc.collect()


if __name__ == "__main__":
    main()
