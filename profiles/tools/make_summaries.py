"""Summarise ncu output into the files bench.py and DESIGN.md cite.

    python profiles/tools/make_summaries.py LAUNCHES_CSV FULL_RAW_CSV TAG

LAUNCHES_CSV: `ncu --metrics gpu__time_duration.sum --csv --log-file` of a
bench command (per-launch, cold-cache, serialised: compare SHARES only).
FULL_RAW_CSV: `ncu -i <full capture> --page raw --csv` of one inner step's
stress, rmap, accel and sweep launches (ncu --set full).

Writes profiles/launches_<TAG>_summary.json, profiles/traffic_<TAG>.json
(DRAM bytes per inner step per kernel class, read by bench.py for
roofline.traffic) and profiles/ncu_full_<TAG>_key.csv (key metrics per
launch).
"""
import csv
import json
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))  # profiles/

CLASS_OF = {"k32_stress_csr": "stress32", "k32_rmap": "stress32", "k32_accel_csr": "accel32",
            "k32_kick_drift": "kick_drift32", "k32_vmax": "reduce32",
            "k_solid_stress": "stress", "k_solid_stress_csr": "stress", "k_solid_rmap": "stress",
            "k_solid_accel": "accel", "k_solid_accel_csr": "accel",
            "k_sweep_tiled": "sweep", "k_sweep_flow": "sweep",
            "k_sweep_tiled32": "sweep32", "k_sweep_flow32": "sweep32",
            "k_solid_kick_drift": "kick_drift", "k_solid_vmax": "reduce", "k_ctrl": "reduce"}
KEY = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "sm__warps_active.avg.pct_of_peak_sustained_active",
       "l1tex__throughput.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
       "lts__throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active"]

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def short(name):
    base = name.split("(")[0].replace("void ", "").replace("mtsph::", "")
    s = base.split("<")[0].strip()
    # the fp32 instantiation of the shared sweep kernels
    return s + "32" if s.startswith("k_sweep") and "float" in base else s


def launch_list(path):
    """[(kernel, ms, segment)] in launch order; a new segment starts at each
    neighbourhood build (its first kernel, k_cell_keys), so the solid
    problem of bench.py is segment 1 and its membrane leg segment 2."""
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    k, m, u, v = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    out, seg, prev = [], 0, None
    for r in rows[hdr_i + 1:]:
        if len(r) <= v or r[m] != "gpu__time_duration.sum":
            continue
        name = short(r[k])
        if name == "k_cell_keys" and prev != "k_cell_keys":
            seg += 1
        prev = name
        out.append((name, float(r[v].replace(",", "")) * SCALE.get(r[u], 1.0), seg))
    return out


def launches(path, segment=None):
    per = {}
    for name, ms, seg in launch_list(path):
        if segment is not None and seg != segment:
            continue
        e = per.setdefault(name, {"launches": 0, "total_ms": 0.0})
        e["launches"] += 1
        e["total_ms"] += ms
    tot = sum(e["total_ms"] for e in per.values())
    for e in per.values():
        e["share"] = e["total_ms"] / tot if tot else 0.0
    return dict(sorted(per.items(), key=lambda kv: -kv[1]["total_ms"]))


def full(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in data:
        rec = {"kernel": short(r[ix["Kernel Name"]])}
        for key in KEY:
            if key not in ix:
                continue
            try:
                val = float(r[ix[key]].replace(",", ""))
            except ValueError:
                continue
            unit = units[ix[key]]
            if key.startswith("dram__bytes"):
                val *= SCALE.get(unit, 1.0)
                unit = "byte"
            elif key == "gpu__time_duration.sum":
                val *= SCALE.get(unit, 1.0)
                unit = "ms"
            rec[key] = val
        out.append(rec)
    return out


LIMIT_UNITS = {"l1_lsu_data_pipe": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
               "fp64_pipe": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
               "issue": "smsp__issue_active.avg.pct_of_peak_sustained_active"}


def limiters(recs, hbm_gbs=None):
    """Busiest unit per kernel class (% of peak, time-weighted over the
    class's launches): the L1/LSU data pipe (global + shared wavefronts), the
    FP64 pipe, instruction issue, and HBM (the class's DRAM bytes over its
    time against MEASURED_PEAKS.json hbm_gbs)."""
    if hbm_gbs is None:
        try:
            hbm_gbs = float(json.load(open(os.path.join(os.path.dirname(HERE), "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            hbm_gbs = 6650.0
    lim = {}
    for rec in recs:
        cls = CLASS_OF.get(rec["kernel"])
        if cls is None:
            continue
        t = float(rec.get("gpu__time_duration.sum", 0.0) or 0.0)
        e = lim.setdefault(cls, {"ms": 0.0, "bytes": 0.0, **{u: 0.0 for u in LIMIT_UNITS}})
        e["ms"] += t
        e["bytes"] += float(rec.get("dram__bytes_read.sum", 0.0) or 0.0) + \
            float(rec.get("dram__bytes_write.sum", 0.0) or 0.0)
        for u, key in LIMIT_UNITS.items():
            e[u] += t * float(rec.get(key, 0.0) or 0.0)
    for cls, e in lim.items():
        for u in LIMIT_UNITS:
            e[u] = round(e[u] / e["ms"], 1) if e["ms"] else 0.0
        e["hbm"] = round(100.0 * e.pop("bytes") / (e["ms"] * 1e-3) / (hbm_gbs * 1e9), 1) if e["ms"] else 0.0
        e["limiter"] = max(list(LIMIT_UNITS) + ["hbm"], key=lambda u: e[u])
    lim["note"] = ("busiest unit per kernel class (% of peak, time-weighted over the class's launches of one "
                   "inner step) from the ncu --set full capture; hbm = DRAM bytes / time against "
                   f"MEASURED_PEAKS.json hbm_gbs ({hbm_gbs:g} GB/s)")
    return lim


def main():
    lpath, fpath, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    summ = {"source": os.path.basename(lpath),
            "note": "ncu gpu__time_duration.sum per launch (cold-cache, serialised, --clock-control none); "
                    "compare shares with bench.py's kernels[*].share, not absolute times",
            "kernels": launches(lpath)}
    # shares within each step variant (the launch list also holds setup,
    # the fp32 variant and the membrane leg)
    solid = launches(lpath, segment=1)
    for tagv, keep in (("fp64_step_shares", lambda k: k.startswith("k_solid_") or k in ("k_sweep_flow", "k_ctrl")),
                       ("fp32_step_shares", lambda k: k.startswith("k32_") or k == "k_sweep_flow32")):
        sel = {k: v["total_ms"] for k, v in solid.items()
               if keep(k) and k not in ("k_solid_gsum", "k_solid_measure", "k32_static", "k32_narrow",
                                        "k32_convert")}
        tot = sum(sel.values())
        summ[tagv] = {k: round(v / tot, 4) for k, v in sorted(sel.items(), key=lambda kv: -kv[1])} if tot else {}
    json.dump(summ, open(os.path.join(HERE, f"launches_{tag}_summary.json"), "w"), indent=1)
    recs = full(fpath)
    traffic = {}
    for rec in recs:
        cls = CLASS_OF.get(rec["kernel"])
        if cls is None:
            continue
        traffic[cls] = traffic.get(cls, 0.0) + rec["dram__bytes_read.sum"] + rec["dram__bytes_write.sum"]
    traffic["note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per inner step for each kernel class "
                       "(one ncu --set full capture of every launch of one step: stress = gather + rmap, "
                       "sweep = all colour launches of both passes); same unit as roofline.achieved x time")
    traffic["source"] = f"ncu_full_{tag}_key.csv"
    json.dump(traffic, open(os.path.join(HERE, f"traffic_{tag}.json"), "w"), indent=1)
    # the unit that limits each kernel class, from the same capture: the
    # busiest of the L1/LSU data pipe (global + shared wavefronts), the FP64
    # pipe, instruction issue and DRAM (time-weighted over the class's launches)
    lim = limiters(recs)
    lim["source"] = f"ncu_full_{tag}_key.csv"
    json.dump(lim, open(os.path.join(HERE, f"limiters_{tag}.json"), "w"), indent=1)
    with open(os.path.join(HERE, f"ncu_full_{tag}_key.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel"] + KEY)
        for rec in recs:
            w.writerow([rec["kernel"]] + [rec.get(k, "") for k in KEY])
    print(json.dumps({k: v for k, v in traffic.items() if not isinstance(v, str)}))


if __name__ == "__main__":
    main()
