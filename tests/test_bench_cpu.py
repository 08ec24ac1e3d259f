"""CPU: the bench.py contract pieces that do not need a GPU.

* the reference arm (`--impl reference`) prints one JSON line with the contract keys;
* the weak-scaling slab builders hand every rank exactly its planes of the global grid
  (a 2-rank config-1 run = one 64^4 replica per rank, slabs stitched = the whole grid);
* our arm fails loudly without a device (no CPU fallback).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json(ref):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "config0",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "impl", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "cpu_baseline", "e2e", "config"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1


def test_weak_scaling_slabs_stitch():
    import workloads
    from paper_2111_11866_b200 import dist as ssd
    world = 2
    whole = workloads.config1(replicas=world)
    parts = []
    for rank in range(world):
        lb, cnt = ssd.partition(64 * world, world)[rank]
        wl = workloads.config1(replicas=world, planes=(lb - 1, lb + cnt))
        assert wl.image.shape[0] == cnt + 2
        # the slab's planes (halos included) equal the whole grid's
        assert np.array_equal(wl.image, whole.image[lb - 1:lb + cnt + 1])
        assert np.array_equal(wl.u0, whole.u0[lb - 1:lb + cnt + 1])
        parts.append(wl.image[1:-1])
    assert np.array_equal(np.concatenate(parts), whole.image[1:-1])


def test_our_arm_needs_a_device():
    import paper_2111_11866_b200 as ss
    if ss.device_available():
        pytest.skip("a GPU is visible")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", "config0", "--steps", "1"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode != 0  # no CPU fallback: the session cannot be created


def test_committed_bench_line_is_consistent():
    """The round's final config-4 line (profiles/, written by bench.py on a B200) carries every
    contract key and its numbers agree with one another: value = doxels x sweeps / time, the
    roofline's achieved = algorithmic bytes per launch / average launch time, frac = achieved /
    peak, the declared copies = 8 B per interior doxel each way."""
    d = json.load(open(os.path.join(ROOT, "profiles", "r02_s5_bench_config4_final.json")))
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "cpu_baseline", "clocks"):
        assert k in d, k
    n = int(np.prod(d["config"]["dims"]))
    assert d["config"]["workload"].startswith("config4") and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert d["sweeps_timed"] == 50 * d["steps"]
    assert d["value"] == pytest.approx(n * d["sweeps_timed"] / (d["ms_per_step"] * d["steps"] * 1e-3), rel=1e-9)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert r["bytes_per_launch"] == 28.0 * n  # 56 B per doxel per red+black sweep, two launches
    assert r["achieved"] == pytest.approx(r["bytes_per_launch"] / (r["avg_launch_ms"] * 1e-3) / 1e9, rel=1e-9)
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-9) and 0.6 < r["frac"] < 0.875
    assert r["traffic"] > r["bytes_per_launch"]  # the two-pass design moves >= 32 B x N per launch
    # the dominant kernel's time fits inside the step
    assert 2 * 50 * r["avg_launch_ms"] < d["ms_per_step"]
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] == 8 * n and 0 < e["value"] < d["value"]
    assert d["gpu_launches"] > 0 and d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
