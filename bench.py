#!/usr/bin/env python
"""Benchmark: inner solid-relaxation particle-steps/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload bar_3d] [--dp 0.02] [--sweep coloured|serial]

One "step" = one inner relaxation step (NeckingProblem.relax_step +
stable_time_step + energy bookkeeping) over every particle of the
workload: kick/drift, deformation-rate gather, F update, J2 return map
(power-law hardening), stress divergence gather, kick, pairwise implicit
damping sweep, reductions and device-side control.

Workload (BASELINE.json configs[2], the 1-GPU case): 3D bar 20 x 2 x 2,
dp 0.02 (1000 x 100 x 100 = 10,000,000 particles), Wendland C2 with
h = 1.3 dp, rho 1, E 200, nu 0.3, power-law hardening s0 = 0.25,
e0 = 0.01, n = 0.2, left end clamped, fp64.  The bar is pre-stretched
uniformly by 0.5 % (4x the yield strain) so the return map runs its
plastic branch, then relaxed by the timed steps.  The state (~10 GB) is
far larger than L2, so no L2 flush is needed between steps.

`value`: device time (CUDA events captured into the step graph) of K
steps with the state resident in HBM.  `e2e`: the same steps driven
through the reference's per-step protocol over the C ABI
(mtsph_solid_stable_dt + mtsph_solid_relax_step: pinned H2D of the step's
control block, D2H of its energy/time-step result each step), wall clock.

--impl reference: the CPU oracle (a C/OpenMP restatement of the
reference's numba loops, oracle/) on a bounded slice of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0
PRESTRAIN = 0.005


_OUT = None   # the real stdout: the JSON line is the only thing written there


def emit(line):
    out = _OUT if _OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def profile_json(stem):
    """The newest committed profile summary profiles/<stem>_rNN.json (ncu
    data cannot be taken inside a timed run)."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"{stem}_r[0-9][0-9].json")))
    if not paths:
        return {}, None
    try:
        return json.load(open(paths[-1])), os.path.basename(paths[-1])
    except Exception:
        return {}, None


def on_chip_roofline(on_chip, kernels, n, sms=148, sm_mhz=1965.0):
    """The neighbour kernels against the L1 / shared-memory data stage
    (128 B per clock per SM, the unit ncu shows them bound by): bytes it must
    move per particle (gathered records, table words, halo records) over the
    class's time, against sms x 128 B x the SM clock."""
    peak = sms * 128 * sm_mhz * 1e6 / 1e9   # GB/s
    out = {"peak": peak, "unit": "GB/s", "per_class": {}}
    tot_b, tot_ms = 0.0, 0.0
    for name, b in on_chip.items():
        ms = kernels[name]["ms_per_step"]
        gbs = b * n / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        out["per_class"][name] = {"bytes_per_particle": b, "achieved": gbs, "frac": gbs / peak}
        tot_b += b
        tot_ms += ms
    out["neighbour_kernels"] = {"bytes_per_particle": tot_b,
                                "achieved": tot_b * n / (tot_ms / 1e3) / 1e9 if tot_ms > 0 else 0.0}
    out["neighbour_kernels"]["frac"] = out["neighbour_kernels"]["achieved"] / peak
    return out


def load_peaks():
    try:
        with open(PEAKS_PATH) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def workload_params(args):
    from paper_2309_04010_b200.config import resolve
    raw = {"scenario": args.workload, "damping_sweep": args.sweep}
    if args.dp:
        raw["dp"] = args.dp
    return resolve(raw).params


def sample_params(params, target_cols):
    """A slice of the workload (same cross-section, shorter length) for the
    CPU baseline: per-particle work is identical."""
    p = dict(params)
    cols = max(int(target_cols), 8)
    p["length"] = cols * p["dp"]
    return p


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ model

def algorithmic_bytes(d, nnz_pp, pairs_pp, groups_pp, sweep="tiled", w=8):
    """Compulsory HBM bytes per particle per step for each kernel class
    (every array element the kernel needs is moved once; the neighbour
    index table counts its true entries).  w: bytes per real (8: fp64,
    4: the fp32 variant).  See DESIGN.md §4."""
    dd = d * d
    vec, ten = w * d, w * dd
    xv = w * (d + 1)                      # reference position + volume
    if sweep == "tiled":
        # v r/w + 1/m, per pair and pass: two 16-bit local ids + coefficient
        sweep_b = 2 * vec + w + 2 * (4 + w) * pairs_pp
    else:
        # v r/w + X|vol + 1/m, per pair and pass: two int32 ids + group pointer
        sweep_b = 2 * vec + xv + w + 2 * (8 * pairs_pp + 8 * groups_pp)
    # fp64: the dF/dt gather streams the stored kernel-gradient magnitude
    # factor of every table entry (8 B; the north star's precomputed kernel
    # gradients in their smallest form) instead of recomputing it
    stored_grad = 8 * nnz_pp if w == 8 else 0.0
    return {
        # v r/w, a, x (displacement in fp32) r/w, flags
        "kick_drift": 2 * vec + vec + 2 * vec + 1,
        # X|V0, v, csr (+ stored gradient magnitudes), B, F r/w, C_p^-1 r/w, alpha r/w, T write
        "stress": xv + vec + 4 * nnz_pp + stored_grad + ten + 2 * ten + 2 * ten + 2 * w + ten,
        # X|V0, T, csr, rho0, flags, mass, v r/w, a write, static sum V gradW
        "accel": xv + ten + 4 * nnz_pp + w + 1 + w + 2 * vec + vec + vec,
        "sweep": sweep_b,
        "reduce": vec,
    }


def outer_bytes(d, nnz_pp):
    """Compulsory HBM bytes per particle of one outer diffusion step
    (PorousProblem.advance_slow: prep, flux, mass, prep, flux, post,
    flux-rate; fp64).  Gathered neighbour fields count once per particle,
    the CSR index 4 B per entry and pass.  See DESIGN.md §4."""
    w, dd = 8, d * d
    xv, vec, ten = w * (d + 1), w * d, w * dd
    idx = 4 * nnz_pp
    prep_a = ten + w + xv + ten + 4 * w + ten      # F, m_l, X|V0, B -> volc sat coeff J, A
    flux = xv + 2 * w + ten + w + idx + vec         # X|V0, sat, volc, A, coeff -> q
    mass = xv + ten + vec + w + 2 * w + 1 + idx     # X|V0, A, q, volc, m_l r/w, flags
    prep = ten + w + xv + 4 * w
    post = w + xv + w + 1 + w + 2 * vec + vec + 4 * w + 2 * vec   # -> pres mix 1/mix rho_l, M, v_l
    frate = xv + ten + 2 * vec + w + idx + vec
    return prep_a + flux + mass + prep + flux + post + frate


def membrane_params(length_factor=1.0):
    """BASELINE configs[3]: the 40 x 40 x 1 cantilever plate (membrane_3d,
    dp 1/22, 17.1 M particles), configs[1] material, wetted top face."""
    from paper_2309_04010_b200.config import resolve
    base = resolve({"scenario": "membrane_3d"}).params
    return resolve({"scenario": "membrane_3d", "damping_sweep": "tiled",
                    "length": base["length"] * length_factor}).params


def membrane_leg(args):
    """Outer-loop diffusion + porous inner relaxation on BASELINE configs[3]
    (the membrane_3d plate, 17.1 M particles; north star item 4)."""
    from paper_2309_04010_b200.scenarios import build_problem, make_policy
    params = membrane_params()
    t0 = time.perf_counter()
    prob = build_problem(params, sweep="tiled")
    setup_s = time.perf_counter() - t0
    pol = make_policy(params, prob.h_min)
    dev, n = prob.dev, prob.lattice.n
    d = prob.lattice.pos.shape[1]
    k_out = max(3, min(args.steps, 10))
    k_in = max(args.steps, 4)
    for _ in range(args.warmup):
        dev.advance_slow(pol.dt_outer, 0.0)
        dev.relax(pol.eta, pol.cfl, -1.0, pol.dt_outer, max_inner=k_in, min_inner=k_in)
    outer_ms = []
    t0 = time.perf_counter()
    for k in range(k_out):
        dev.advance_slow(pol.dt_outer, (k + 1) * pol.dt_outer)
        outer_ms.append(dev.outer_ms())
    outer_wall = (time.perf_counter() - t0) / k_out
    t0 = time.perf_counter()
    r = dev.relax(pol.eta, pol.cfl, -1.0, pol.dt_outer, max_inner=k_in, min_inner=k_in)
    inner_s = time.perf_counter() - t0
    ms = float(np.mean(outer_ms))
    nnz_pp = dev.sizes()["nnz"] / n
    model = outer_bytes(d, nnz_pp)
    peak, _ = load_peaks()
    out = {"workload": f"membrane_3d plate (BASELINE configs[3]) {params['length']:g} x "
                       f"{params['breadth']:g} x {params['thickness']:g}, dp 1/22 ({n} particles), "
                       "top face wetted, left edge clamped, tiled sweep, fp64",
           "particles": n, "setup_s": setup_s,
           "inner": {"value": n * int(r.n_inner) / inner_s, "unit": "particle-steps/s",
                     "ms_per_step": 1e3 * inner_s / max(int(r.n_inner), 1),
                     "timing": "wall clock around the device loop (graph chunks)"},
           "outer_diffusion": {"value": n / (ms / 1e3), "unit": "particle-steps/s",
                               "ms_per_step": ms, "wall_ms_per_step": 1e3 * outer_wall,
                               "timing": "CUDA events around the 7 kernels of advance_slow"}}
    gbs = model * n / (ms / 1e3) / 1e9
    out["outer_diffusion"].update({"bytes_per_particle": model, "achieved_gbs": gbs,
                                   "frac_of_hbm_peak": gbs / peak,
                                   "neighbours_per_particle": nnz_pp})
    return out


def build_solid(params, sweep):
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.device import DeviceSolid
    from paper_2309_04010_b200.scenarios import _necking_materials
    lat = lattices.build_lattice(params)
    elastic, hard = _necking_materials(params)
    law, hp = hard.device_params()
    t0 = time.perf_counter()
    dev = DeviceSolid(lat.pos, lat.vol, elastic.density0, lat.constrained, lat.side, lat.mid_mask,
                      lat.h_axes, elastic.shear_modulus, elastic.bulk_modulus, plastic=True,
                      hardening_law=law, hard=hp, sweep=sweep)
    setup_s = time.perf_counter() - t0
    d = lat.pos.shape[1]
    nu = elastic.poisson_ratio
    Fm = np.eye(d)
    Fm[0, 0] = 1.0 + PRESTRAIN
    for k in range(1, d):
        Fm[k, k] = 1.0 - nu * PRESTRAIN
    dev.set("F", np.broadcast_to(Fm, (lat.n, d, d)))
    dev.set("pos", lat.pos @ Fm.T)
    return dev, lat, elastic, setup_s


def run_ours(args):
    import torch  # noqa: F401  (plumbing only: torch.distributed for N > 1)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    decomposed = args.mode == "decomposed" or (args.mode == "auto" and world > 1)
    if world > 1 or decomposed:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2309_04010_b200.device import select_device
    select_device(local)                     # the library has its own CUDA runtime
    if decomposed:
        return run_decomposed(args, world, rank, local)
    params = workload_params(args)
    dev, lat, elastic, setup_s = build_solid(params, args.sweep)
    eta, cfl = params["eta"], params["cfl"]
    n, d = lat.pos.shape
    sz = dev.sizes()
    # warm-up (captures the step graph; at least W steps)
    done = 0
    while done < args.warmup:
        dev.run_steps(args.steps, eta, cfl)
        done += args.steps
    launches0 = dev.launches()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    timing = dev.run_steps(args.steps, eta, cfl)
    clk = clocks.stop()
    launches = dev.launches() - launches0
    ms = timing["total_ms"]
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * n * args.steps / (ms / 1e3)
    # end to end through the per-step protocol (host round trip per step)
    e2e_steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        dt = dev.stable_dt(cfl)
        dev.relax_step(dt, eta)
    e2e_s = time.perf_counter() - t0
    e2e = world * n * e2e_steps / e2e_s
    # sizeof(Ctrl) (csrc/damping.cuh): 14 doubles, 4 int64, 4 int, 2 uint64;
    # per step stable_dt + relax_step move it 2x host->device, 4x back
    ctrl_bytes = 14 * 8 + 4 * 8 + 4 * 4 + 2 * 8
    # roofline of the dominant kernel class
    peak, peak_kind = load_peaks()
    model = algorithmic_bytes(d, sz["nnz"] / n, sz["npairs"] / n, sz["ngroups"] / n, args.sweep)
    classes = {"kick_drift": timing["kick_drift_ms"], "stress": timing["stress_ms"],
               "accel": timing["accel_ms"], "sweep": timing["sweep_ms"],
               "reduce": timing["reduce_ms"]}
    kernels = {}
    for name, tms in classes.items():
        per_step_s = tms / 1e3 / args.steps
        gbs = model[name] * n / per_step_s / 1e9 if per_step_s > 0 else 0.0
        kernels[name] = {"ms_per_step": tms / args.steps, "share": tms / ms if ms else 0.0,
                         "bytes_per_particle": model[name], "achieved_gbs": gbs}
    kernels["stress"]["of_which_stored_gradient_magnitudes"] = 8 * sz["nnz"] / n
    # the neighbour kernels' real bound: the SM's L1 / shared-memory data
    # stage (128 B per clock per SM).  Bytes it must move per particle: the
    # gathered records (64 B dF/dt, 96 B divergence) and table words per
    # neighbour visit; per pair update of the sweep (two passes) the 12 B
    # ring entry and both halo records read and written (4 x 32 B)
    nnz_pp, pairs_pp = sz["nnz"] / n, sz["npairs"] / n
    on_chip = {"stress": (64 + 4 + 8) * nnz_pp, "accel": (96 + 4) * nnz_pp,
               "sweep": 2 * (12 + 4 * 32) * pairs_pp}
    top = max(classes, key=classes.get)
    k_top = kernels[top]
    step_bytes = sum(model[k] for k in classes)
    step_gbs = step_bytes * n / (ms / 1e3 / args.steps) / 1e9
    tr, tsrc = profile_json("traffic")
    traffic = tr.get(top)
    lim, lsrc = profile_json("limiters")
    variants = {}
    if not args.no_fp32 and args.sweep == "tiled":
        variants["fp32"] = fp32_variant(dev, args, params, n, d, sz, world, peak)
    if not args.no_serial and args.sweep == "tiled" and world == 1:
        variants["serial"] = serial_variant(params, args)
    line = {
        "metric": "inner solid-relaxation particle-steps/sec",
        "value": value, "unit": "particle-steps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload} (BASELINE configs[2])",
                   "particles_per_gpu": n, "dp": params["dp"], "h_over_dp": params["h_factor"],
                   "material": "rho 1, E 200, nu 0.3, J2 power-law s0 0.25 e0 0.01 n 0.2",
                   "prestrain": PRESTRAIN, "damping_sweep": args.sweep,
                   "sweep_phases": sz["phases"], "neighbours_per_particle": sz["nnz"] / n,
                   "pairs": sz["npairs"], "groups": sz["ngroups"],
                   "l2": "state >> 126 MB L2 (no flush needed)",
                   "parallelism": "1 GPU",
                   "setup_s": setup_s},
        "e2e": {"value": e2e, "unit": "particle-steps/s", "h2d_bytes_per_step": 2 * ctrl_bytes,
                "d2h_bytes_per_step": 4 * ctrl_bytes,
                "path": "C ABI per-step protocol mtsph_solid_stable_dt + mtsph_solid_relax_step"},
        "roofline": {"kernel": top, "bound": "hbm", "achieved": k_top["achieved_gbs"],
                     "peak": peak, "unit": "GB/s",
                     "frac": k_top["achieved_gbs"] / peak, "traffic": traffic,
                     "traffic_source": tsrc,
                     "whole_step": {"bytes_per_particle": step_bytes, "achieved": step_gbs,
                                    "frac": step_gbs / peak},
                     "on_chip_data_stage": on_chip_roofline(on_chip, kernels, n),
                     "limiter": (lim.get(top) or {}).get("limiter"),
                     "limiter_pct_of_peak": {k: v for k, v in (lim.get(top) or {}).items()
                                             if k not in ("ms", "limiter")},
                     "limiter_source": lsrc,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
        "kernels": kernels,
        "variants": variants,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if not args.no_membrane and world == 1:
        del dev
        line["membrane"] = membrane_leg(args)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(params, args, budget_s=args.cpu_budget)
    if rank == 0:
        emit(line)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def serial_variant(params, args):
    """Parity mode at full size: the same workload with the reference's exact
    damping order (bit-identical to the serial sequence, the multi-CTA
    level-scheduled kernel), a few steps timed the same way."""
    t0 = time.perf_counter()
    dev, lat, _, _ = build_solid(params, "serial")
    setup = time.perf_counter() - t0
    eta, cfl = params["eta"], params["cfl"]
    steps = max(2, min(args.steps, 5))
    dev.run_steps(1, eta, cfl)
    t = dev.run_steps(steps, eta, cfl)
    sz = dev.sizes()
    out = {"damping_order": "serial (the reference's exact order; multi-CTA level-scheduled kernel)",
           "value": lat.n * steps / (t["total_ms"] / 1e3), "unit": "particle-steps/s",
           "ms_per_step": t["total_ms"] / steps, "sweep_ms_per_step": t["sweep_ms"] / steps,
           "levels": sz["phases"], "groups": sz["ngroups"], "steps": steps, "setup_s": setup,
           "finite": dev.measure()["finite"]}
    del dev
    return out


def fp32_variant(dev, args, params, n, d, sz, world, peak):
    """The north star's separately reported fp32 variant: the same solid
    switched to single-precision state (csrc/solid32.cuh), same steps."""
    eta, cfl = params["eta"], params["cfl"]
    dev.set_precision(32)
    done = 0
    while done < args.warmup:
        dev.run_steps(args.steps, eta, cfl)
        done += args.steps
    timing = dev.run_steps(args.steps, eta, cfl)
    ms = timing["total_ms"]
    if world > 1:
        import torch
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    fin = dev.measure()["finite"]
    dev.set_precision(64)
    model = algorithmic_bytes(d, sz["nnz"] / n, sz["npairs"] / n, sz["ngroups"] / n, "tiled", w=4)
    kernels = {}
    for name in ("kick_drift", "stress", "accel", "sweep", "reduce"):
        tms = timing[name + "_ms"]
        per_step_s = tms / 1e3 / args.steps
        gbs = model[name] * n / per_step_s / 1e9 if per_step_s > 0 else 0.0
        kernels[name] = {"ms_per_step": tms / args.steps, "share": tms / ms if ms else 0.0,
                         "bytes_per_particle": model[name], "achieved_gbs": gbs}
    top = max(kernels, key=lambda k: kernels[k]["ms_per_step"])
    return {"dtype": "f32 (state, gathers, sweep; return map evaluated in f64)",
            "value": world * n * args.steps / (ms / 1e3), "unit": "particle-steps/s",
            "ms_per_step": ms / args.steps, "finite": fin,
            "roofline": {"kernel": top, "bound": "hbm", "achieved": kernels[top]["achieved_gbs"],
                         "peak": peak, "unit": "GB/s",
                         "frac": kernels[top]["achieved_gbs"] / peak},
            "kernels": kernels}


def scale_params(args, world):
    """BASELINE configs[4]: the seeded +-5 % jittered power-law block
    (config-0 material, dp 0.02, 2 x 2 cross-section = 100 x 100 particles),
    lengthened along x to the requested count: 32 M particles split over the
    N GPUs (strong scaling) or 4 M per GPU (weak scaling)."""
    from paper_2309_04010_b200.config import resolve
    if args.scaling == "strong":
        total = args.scale_particles or 32e6
    else:
        total = (args.scale_particles or 4e6) * world
    base = resolve({"scenario": "block_3d", "damping_sweep": "tiled"}).params
    per_col = round(base["width"] / base["dp"]) * round(base["breadth"] / base["dp"])
    cols = max(int(round(total / per_col)), 8)
    return resolve({"scenario": "block_3d", "damping_sweep": "tiled",
                    "length": cols * base["dp"]}).params


def run_decomposed(args, world, rank, local):
    """N > 1 (or --mode decomposed): BASELINE configs[4] split into N x-slabs
    (partition.py), one per GPU, halo exchanges over NCCL each phase, rank
    reductions all-gathered on the device and the stopping rule applied by
    every rank's control kernel (DecomposedSolid.relax_device).  --scaling
    strong (default): the 32 M-particle block split N ways; weak: 4 M
    particles per GPU (the block N times longer)."""
    import torch
    import torch.distributed as dist
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.distributed import DecomposedSolid
    from paper_2309_04010_b200.scenarios import _necking_materials
    from paper_2309_04010_b200.config import resolve
    params = scale_params(args, world)
    lat = lattices.build_lattice(params)
    elastic, hard = _necking_materials(params)
    eta, cfl = params["eta"], params["cfl"]
    t0 = time.perf_counter()
    dec = DecomposedSolid(lat, elastic, hard, world, ranks=[rank], group="torch", dist=dist,
                          tensor_device=f"cuda:{local}")
    setup_s = time.perf_counter() - t0
    dev = dec.devices[0]
    plan = dec.plans[rank]
    d = lat.pos.shape[1]
    Fm = np.eye(d)
    Fm[0, 0] = 1.0 + PRESTRAIN
    for k in range(1, d):
        Fm[k, k] = 1.0 - elastic.poisson_ratio * PRESTRAIN
    dev.set("F", np.broadcast_to(Fm, (len(plan.local_ids), d, d)))
    dev.set("pos", lat.pos[plan.local_ids] @ Fm.T)
    n_total = lat.n
    n_own = int((~plan.ghost).sum())
    stream = torch.cuda.ExternalStream(dev.stream_handle())
    dec.relax_device(eta, cfl, -1.0, 1.0, fixed_steps=max(args.warmup, 3), check_every=max(args.warmup, 3))
    launches0 = dev.launches()
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dec.issue_s, dec.issue_steps, replays0 = 0.0, 0, dec.graph_replays
    e0.record(stream)
    dec.relax_device(eta, cfl, -1.0, 1.0, fixed_steps=args.steps, check_every=args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    # kernels of replayed steps are launched by the graph, not counted by the library
    launches = dev.launches() - launches0 + (dec.graph_replays - replays0) * dec.graph_launches
    host_issue_ms = 1e3 * dec.issue_s / max(dec.issue_steps, 1)
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    # end to end: the host-controlled decomposed loop (per-phase reductions
    # read back to the host, exchanges as above), wall clock, max over ranks
    e2e_steps = max(3, min(args.steps, 10))
    dist.barrier()
    w0 = time.perf_counter()
    dec.relax(eta, cfl, -1.0, 1.0, fixed_steps=e2e_steps)
    torch.cuda.synchronize()
    wall = torch.tensor([time.perf_counter() - w0], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(wall, op=dist.ReduceOp.MAX)
    counts = torch.tensor([n_own, len(plan.local_ids) - n_own], dtype=torch.float64,
                          device=f"cuda:{local}")
    dist.all_reduce(counts)
    line = {
        "metric": "inner solid-relaxation particle-steps/sec",
        "value": n_total * args.steps / (ms / 1e3), "unit": "particle-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"block_3d (BASELINE configs[4], jittered +-5 %, seed "
                               f"{params['seed']}), {args.scaling} scaling",
                   "particles": n_total, "particles_per_gpu": n_total // world,
                   "dp": params["dp"], "h_over_dp": params["h_factor"],
                   "material": "rho 1, E 200, nu 0.3, J2 power-law s0 0.25 e0 0.01 n 0.2",
                   "prestrain": PRESTRAIN, "damping_sweep": "tiled",
                   "parallelism": f"{world} x-slabs, one GPU each; NCCL halo exchange per phase "
                                  "(grouped send/recv), device-side control (all-gather)",
                   "ghost_particles_total": int(counts[1].item()),
                   "step_issue": "CUDA graph replay (phases + NCCL exchanges + control captured once)"
                                 if dec._graph else "eager enqueue from Python",
                   "host_issue_ms_per_step": host_issue_ms,
                   "l2": "state >> 126 MB L2 (no flush needed)", "setup_s": setup_s,
                   "timing": "CUDA events on each rank's solid stream around the enqueued "
                             "steps; max over ranks"},
        "e2e": {"value": n_total * e2e_steps / float(wall.item()), "unit": "particle-steps/s",
                "h2d_bytes_per_step": 8 * 8, "d2h_bytes_per_step": 8 * 4 * (2 + 2 * dec.ncolours),
                "path": "host-controlled decomposed loop (DecomposedSolid.relax): per-phase "
                        "reductions read back to the host, wall clock, max over ranks"},
        "gpu_launches": launches,
        "clocks": clk,
    }
    # roofline of the whole per-rank step (the decomposed loop has no
    # per-class events): algorithmic bytes of every class for the rank's
    # owned particles over the step time
    sz = dev.sizes()
    nl = len(plan.local_ids)
    model = algorithmic_bytes(d, sz["nnz"] / nl, sz["npairs"] / nl, sz["ngroups"] / nl, "tiled")
    peak, peak_kind = load_peaks()
    gbs = sum(model.values()) * (n_total / world) / (ms / args.steps / 1e3) / 1e9
    line["roofline"] = {"kernel": "whole inner step per rank", "bound": "hbm", "achieved": gbs,
                        "peak": peak, "unit": "GB/s", "frac": gbs / peak, "traffic": None,
                        "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"}
    del dec, dev
    if not args.no_membrane:
        try:
            line["membrane"] = membrane_decomposed(args, world, rank, local)
        except Exception as e:   # the solid line above stands on its own
            line["membrane"] = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        emit(line)
    dist.destroy_process_group()


def membrane_decomposed(args, world, rank, local):
    """BASELINE configs[3] on N GPUs: the membrane_3d plate (17.1 M
    particles split N ways; --scaling weak: the plate N times longer) on
    x-slabs, porous inner steps device-controlled (DecomposedPorous.
    relax_device, NCCL halos and all-gather), one outer diffusion step with
    its exchanges."""
    import torch
    import torch.distributed as dist
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.config import resolve
    from paper_2309_04010_b200.distributed import DecomposedPorous
    from paper_2309_04010_b200.scenarios import _membrane, make_policy
    params = membrane_params(world if args.scaling == "weak" else 1)
    lat = lattices.build_lattice(params)
    pol = make_policy(params, float(np.min(lat.h_axes)))
    t0 = time.perf_counter()
    dec = DecomposedPorous(lat, _membrane(params), params["contact_time"],
                           params["evaporation_rate"], world, ranks=[rank], group="torch",
                           dist=dist, tensor_device=f"cuda:{local}")
    setup_s = time.perf_counter() - t0
    dev = dec.devices[0]
    stream = torch.cuda.ExternalStream(dev.stream_handle())
    k_in = max(args.steps, 4)
    dec.advance_slow(pol.dt_outer, pol.dt_outer)
    dec.relax_device(pol.eta, pol.cfl, -1.0, pol.dt_outer, fixed_steps=3, check_every=3)
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    dec.relax_device(pol.eta, pol.cfl, -1.0, pol.dt_outer, fixed_steps=k_in, check_every=k_in)
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    inner_ms = float(t.item()) / k_in
    dist.barrier()
    w0 = time.perf_counter()
    dec.advance_slow(pol.dt_outer, 2 * pol.dt_outer)
    torch.cuda.synchronize()
    w = torch.tensor([time.perf_counter() - w0], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(w, op=dist.ReduceOp.MAX)
    n = lat.n
    return {"workload": f"membrane_3d plate (BASELINE configs[3]) {params['length']:g} x "
                        f"{params['breadth']:g} x {params['thickness']:g} ({n} particles, "
                        f"{n // world} per GPU), tiled sweep, fp64, {world} x-slabs",
            "setup_s": setup_s,
            "inner": {"value": n / (inner_ms / 1e3), "unit": "particle-steps/s",
                      "ms_per_step": inner_ms,
                      "timing": "CUDA events on each rank's stream around the device-controlled "
                                "steps; max over ranks"},
            "outer_diffusion": {"value": n / float(w.item()), "unit": "particle-steps/s",
                                "ms_per_step": 1e3 * float(w.item()),
                                "timing": "wall clock of one outer step (host-synchronised "
                                          "phases and exchanges); max over ranks"}}


def cpu_baseline(params, args, budget_s=20.0, steps=None):
    """Oracle (C/OpenMP restatement of the reference loops) on a slice."""
    from oracle import oracle as O
    from oracle.problems import NeckingOracle
    from paper_2309_04010_b200 import lattices
    from paper_2309_04010_b200.scenarios import _necking_materials
    sp = sample_params(params, args.cpu_cols)
    lat = lattices.build_lattice(sp)
    elastic, hard = _necking_materials(sp)
    law, hd = hard.device_params()
    t0 = time.perf_counter()
    prob = NeckingOracle(lat.pos, lat.vol, elastic.density0, lat.constrained,
                         lat.side < 0, lat.side > 0, lat.mid_mask, elastic.shear_modulus,
                         elastic.bulk_modulus, hd, float(lat.h_axes[0]), hardening_law=law)
    build_s = time.perf_counter() - t0
    d = lat.pos.shape[1]
    Fm = np.eye(d)
    Fm[0, 0] = 1.0 + PRESTRAIN
    for k in range(1, d):
        Fm[k, k] = 1.0 - elastic.poisson_ratio * PRESTRAIN
    prob.F[:] = Fm
    prob.pos[:] = lat.pos @ Fm.T
    n = lat.n
    done, t0 = 0, time.perf_counter()
    while True:
        dt = prob.stable_time_step(params["cfl"])
        prob.relax_step(dt, params["eta"])
        done += 1
        el = time.perf_counter() - t0
        if (steps is not None and done >= steps) or (steps is None and el > budget_s):
            break
    return {"value": n * done / el, "unit": "particle-steps/s", "cores": O.lib().or_num_threads(),
            "kind": "port",
            "sample": f"{args.workload} slice {sp['length']:g} x {sp['width']:g} x "
                      f"{sp['breadth']:g} ({n} particles), {done} inner steps in {el:.1f} s "
                      f"(oracle build {build_s:.1f} s excluded); serial damping sweep"}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # rank 0 alone does the work, with every host thread (torchrun exports
    # OMP_NUM_THREADS=1 to each rank)
    from oracle import oracle as O
    O.lib().or_set_num_threads(len(os.sched_getaffinity(0)))
    params = workload_params(args)
    steps = max(args.steps, 1)
    base = cpu_baseline(params, args, steps=steps + args.warmup)
    line = {
        "impl": "reference", "metric": "inner solid-relaxation particle-steps/sec",
        "value": base["value"], "unit": "particle-steps/s", "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload} (BASELINE configs[2])", "dp": params["dp"]},
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "particle-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="bar_3d")
    ap.add_argument("--dp", type=float, default=0.0)
    ap.add_argument("--sweep", default="tiled", choices=("tiled", "coloured", "serial"))
    ap.add_argument("--cpu-cols", type=int, default=10)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the fp32 variant")
    ap.add_argument("--no-serial", action="store_true",
                    help="skip the reference-order (parity mode) variant")
    ap.add_argument("--mode", default="auto", choices=("auto", "decomposed"),
                    help="auto: N = 1 single domain, N > 1 slab decomposition with NCCL halos; "
                         "decomposed forces the decomposed path (also at N = 1)")
    ap.add_argument("--scaling", default="strong", choices=("weak", "strong"),
                    help="decomposed runs (BASELINE configs[4], the jittered power-law "
                         "block): strong = 32 M particles split N ways, weak = 4 M per GPU")
    ap.add_argument("--scale-particles", type=float, default=0.0,
                    help="decomposed runs: total (strong) or per-GPU (weak) particle count; "
                         "default 32e6 / 4e6")
    ap.add_argument("--no-membrane", action="store_true", help="skip the porous membrane leg")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun
        # (127.0.0.1 rendezvous); the ranks see WORLD_SIZE and do not recurse
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; "
                         "launch with matching --nproc-per-node")
    # keep stdout for the JSON line alone: library output on fd 1 (NCCL's
    # version banner, ...) goes to stderr
    global _OUT
    _OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
