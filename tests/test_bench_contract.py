"""bench.py's JSON contract, checked on CPU with the reference arm at config 1.

The GPU arm is exercised on a B200 (the driver's round-end bench); here the
reference arm (the CPU oracle, the only thing that runs without a GPU) must
print exactly one JSON line with the keys the driver reads.
"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_reference_arm_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "voxel/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["metric"] == bench.METRIC
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": "voxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_workloads_cover_the_baseline_configs():
    # BASELINE.json configs 1-5, each with a bounded CPU sample
    assert {"c1", "c2", "c3", "c4", "c5"} <= set(bench.WORKLOADS)
    for name, wl in bench.WORKLOADS.items():
        assert len(wl["brick"]) == len(wl["shape"]) and wl["levels"] >= 1 and wl["desc"]
        s = wl["sample"]
        assert len(s["shape"]) == len(wl["shape"]) and s["levels"] <= wl["levels"]
    assert bench.WORKLOADS["c5"]["timesteps"] == 16
    assert bench.ALG_BYTES_PER_UNKNOWN_ITER == {3: 56, 2: 52}


def test_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun starts two ranks itself (one process per GPU; gloo on CPU)
    whose communicator really has two members."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-probe"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT,
                         env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = lines[0]
    assert d["n_gpus"] == 2 and d["comm"]["nranks"] == 2 and d["comm"]["all_reduce_ok"] is True


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-probe"],
                         capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode == 2 and "WORLD_SIZE" in out.stderr
