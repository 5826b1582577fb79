"""Per-step cost of the reference-order (serial) damping sweep at benchmark
scale: the multi-CTA kernel (MTSPH_SERIAL_GRID=1), the one-CTA global
kernel (only where it finishes in reasonable time) and the tiled order, on
slices of the BASELINE configs[2] bar (same cross-section, growing length).
Device time from the step graph's CUDA events (run_steps).

    python profiles/tools/serial_scale_probe.py --lengths 0.2,1,4,20 > profiles/serial_scale_r02.jsonl
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lengths", default="0.2,1,4,20")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--one-cta-max", type=float, default=1.0,
                    help="largest bar length timed with the one-CTA kernel")
    args = ap.parse_args()
    for length in [float(x) for x in args.lengths.split(",")]:
        modes = [("serial multi-CTA", "serial", "1"), ("tiled", "tiled", "0")]
        if length <= args.one_cta_max:
            modes.insert(1, ("serial one-CTA", "serial", "0"))
        for label, sweep, grid in modes:
            os.environ["MTSPH_SERIAL_GRID"] = grid
            a = argparse.Namespace(workload="bar_3d", sweep=sweep, dp=0.0)
            params = dict(bench.workload_params(a))
            params["length"] = length
            t0 = time.perf_counter()
            dev, lat, _, _ = bench.build_solid(params, sweep)
            setup = time.perf_counter() - t0
            dev.run_steps(2, params["eta"], params["cfl"])
            t = dev.run_steps(args.steps, params["eta"], params["cfl"])
            sz = dev.sizes()
            print(json.dumps({"length": length, "particles": lat.n, "sweep": label,
                              "levels_or_phases": sz["phases"], "groups": sz["ngroups"],
                              "ms_per_step": t["total_ms"] / args.steps,
                              "sweep_ms": t["sweep_ms"] / args.steps,
                              "setup_s": round(setup, 1)}), flush=True)
            del dev


if __name__ == "__main__":
    main()
