"""CPU: the benchmark's byte models and the profile summariser (host logic
behind bench.py's roofline and profiles/launches_*_summary.json)."""

import os
import sys

from conftest import ROOT

sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "profiles", "tools"))


def test_algorithmic_bytes_fp64_and_fp32():
    import bench
    m64 = bench.algorithmic_bytes(3, 78.37, 39.19, 39.19, "tiled", w=8)
    m32 = bench.algorithmic_bytes(3, 78.37, 39.19, 39.19, "tiled", w=4)
    # the sweep: v r/w + 1/m + (2 x 16-bit ids + coefficient) per pair and pass
    assert abs(m64["sweep"] - (2 * 24 + 8 + 2 * 12 * 39.19)) < 1e-9
    assert abs(m32["sweep"] - (2 * 12 + 4 + 2 * 8 * 39.19)) < 1e-9
    for k in ("kick_drift", "stress", "accel", "reduce"):
        assert m32[k] < m64[k]
    # the index table (4 B per neighbour) is the same in both precisions
    assert m64["stress"] - m32["stress"] > 0
    assert abs((m64["accel"] - m32["accel"]) - (4 * 4 + 4 * 9 + 4 + 4 + 4 * 3 * 4)) < 1e-9


def test_on_chip_roofline_accounts_per_class_and_total():
    import bench
    k = {"stress": {"ms_per_step": 4.0}, "accel": {"ms_per_step": 5.0}, "sweep": {"ms_per_step": 6.0}}
    oc = {"stress": 6000.0, "accel": 8000.0, "sweep": 11000.0}
    r = bench.on_chip_roofline(oc, k, 10_000_000)
    assert abs(r["peak"] - 148 * 128 * 1.965) < 1e-6          # GB/s
    assert abs(r["per_class"]["accel"]["achieved"] - 8000.0 * 1e7 / 5e-3 / 1e9) < 1e-6
    tot = r["neighbour_kernels"]
    assert abs(tot["achieved"] - 25000.0 * 1e7 / 15e-3 / 1e9) < 1e-6
    assert 0 < tot["frac"] < 1


def test_outer_bytes_counts_index_per_gather_pass():
    import bench
    a, b = bench.outer_bytes(3, 70.0), bench.outer_bytes(3, 71.0)
    assert abs((b - a) - 4 * 4) < 1e-9          # flux x 2, mass, flux rate


def test_launch_list_segments(tmp_path):
    import make_summaries as ms
    hdr = '"ID","Kernel Name","Metric Name","Metric Unit","Metric Value"\n'
    rows = ["k_cell_keys", "void k_solid_stress_csr<3, 4>(SolidArgs)", "k_sweep_flow<3, double>(x)",
            "k_sweep_flow<3, float>(x)", "k_cell_keys", "void k_por_accel<3>(PorousArgs)"]
    text = hdr + "".join(f'"{i}","{k}","gpu__time_duration.sum","ms","1.5"\n' for i, k in enumerate(rows))
    p = tmp_path / "l.csv"
    p.write_text(text)
    L = ms.launch_list(str(p))
    assert [seg for _, _, seg in L] == [1, 1, 1, 1, 2, 2]
    assert [k for k, _, _ in L][2:4] == ["k_sweep_flow", "k_sweep_flow32"]
    solid = ms.launches(str(p), segment=1)
    assert set(solid) == {"k_cell_keys", "k_solid_stress_csr", "k_sweep_flow", "k_sweep_flow32"}
    assert abs(sum(v["share"] for v in solid.values()) - 1.0) < 1e-12


def test_bench_gpus_n_launches_n_ranks():
    """`bench.py --gpus 2` started without torchrun re-launches itself as two
    ranks (127.0.0.1 rendezvous); the reference arm runs on rank 0 alone with
    every host thread and reports n_gpus 2.  (The GPU arm's ranks are the
    same launch; it needs the GPUs.)"""
    import json
    import subprocess
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--impl", "reference", "--steps", "1", "--warmup", "3",
                          "--cpu-cols", "8"], capture_output=True, text=True, env=env,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["n_gpus"] == 2
    assert rec["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


def test_bench_rejects_mismatched_world_size():
    import subprocess
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--impl", "reference"], capture_output=True, text=True, env=env,
                         timeout=300, cwd=ROOT)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
