"""Tuning sweep (GPU): tiled-sweep block size (MTSPH_TILE_BITS) and CTA
size (MTSPH_TILE_THREADS); one solid per setting, both precisions.

    python profiles/tools/tune_sweep.py --cases 6:0,7:0,7:1024,6:512:448
    (bits:threads[:sub-colour cap]; MTSPH_LIB selects a tuning build)
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
    ap.add_argument("--cases", default="6:0,7:0")
    args = ap.parse_args()
    params = bench.workload_params(args)
    eta, cfl = params["eta"], params["cfl"]
    for case in args.cases.split(","):
        bits, th, *rest = case.split(":")
        os.environ["MTSPH_TILE_BITS"] = bits
        if rest:
            os.environ["MTSPH_SWEEP_SUBCAP"] = rest[0]
        else:
            os.environ.pop("MTSPH_SWEEP_SUBCAP", None)   # the schedule's default
        if th != "0":
            os.environ["MTSPH_TILE_THREADS"] = th
        else:
            os.environ.pop("MTSPH_TILE_THREADS", None)
        try:
            dev, lat, _, setup = bench.build_solid(params, args.sweep)
        except Exception as e:  # a block that does not fit shared memory
            print(case, "failed:", e, flush=True)
            continue
        for bits_p in (64, 32):
            dev.set_precision(bits_p)
            dev.run_steps(args.steps, eta, cfl)
            t = dev.run_steps(args.steps, eta, cfl)
            out = {k: round(v / args.steps, 3) for k, v in t.items() if k.endswith("_ms")}
            print(f"case={case} fp{bits_p}", json.dumps(out), "setup", round(setup, 1),
                  flush=True)
        del dev


if __name__ == "__main__":
    main()
