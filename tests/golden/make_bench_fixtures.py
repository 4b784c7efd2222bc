"""Frozen oracle fixtures for the BENCHMARKED configurations at full size (run in the build container).

    python tests/golden/make_bench_fixtures.py [c4] [c3] [c5]

The random walker has no reference implementation, so these are outputs of the float64
oracle (`oracle.rw`, tol 1e-10), on exactly the inputs `bench.py` segments — the §8(d) generator
(`synthetic.phantom_streamed`, bit-identical to `synthetic.phantom` = `default_rng(0xC0FFEE)`):

* `c4_top.npz` — config 4 (1024^3, 32^3 bricks, 4 levels, seeds S1): SHA-256 of every LOD level and
  projected seed level (the oracle's; the GPU LOD must reproduce them bit for bit), and the oracle's
  whole-level solve of the 128^3 coarsest level (every 2nd voxel per axis).
* `c3_top.npz` — config 3 (16384^2, 64^2 tiles, 9 levels): the same, coarsest level 64^2 (full).
* `c5_top.npz` — config 5 (512^3 x 16 timesteps, per-timestep 4-level hierarchy): timesteps
  0, 7 and 15 (`synthetic.series_timestep`), coarsest 64^3 levels (every 2nd voxel per axis).

The finer levels are checked in the GPU tests (`tests/test_bench_configs.py`) brick by brick: a fixed
random sample of bricks per level is solved by the oracle from the GPU's own parent level
(`oracle.rw.solve_brick`) — the full-size finer levels would take the float64 oracle hours.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import lod, rw  # noqa: E402
from paper_2509_26213_b200 import synthetic as syn  # noqa: E402

TOP = rw.RWParams(beta=100.0, min_weight=1e-6, tol=1e-10, max_iter=100_000)
BENCH = {
    "c4": dict(shape=(1024, 1024, 1024), brick=(32, 32, 32), levels=4, seeds="S1", stride=2),
    "c3": dict(shape=(16384, 16384), brick=(64, 64), levels=9, seeds="S1", stride=1),
    "c5": dict(shape=(512, 512, 512), brick=(32, 32, 32), levels=4, seeds="S1", stride=2, timesteps=16,
               sampled_t=(0, 7, 15)),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def pyramid(vol, seeds, levels):
    vols, sds = [vol], [seeds]
    for _ in range(levels - 1):
        vols.append(lod.lod_down_slabbed(vols[-1]))
        sds.append(rw.project_seeds(sds[-1]))
    return vols, sds


def top_fixture(vol, seeds, spec, prefix, out, meta):
    t0 = time.time()
    vols, sds = pyramid(vol, seeds, spec["levels"])
    res = rw.solve_level(vols[-1], sds[-1], vols[-1].shape, None, TOP)
    s = spec["stride"]
    sub = tuple(slice(None, None, s) for _ in vols[-1].shape)
    out[f"{prefix}top_prob"] = res.prob[sub].astype(np.float32)
    meta[prefix or "top"] = {
        "volume_sha256": [sha(v) for v in vols], "seeds_sha256": [sha(x) for x in sds],
        "top_shape": list(vols[-1].shape), "top_iterations": int(res.iterations.max()),
        "top_converged": bool(res.converged.all()), "seconds": round(time.time() - t0, 1)}
    print(prefix, meta[prefix or "top"], flush=True)


def make(name):
    spec = BENCH[name]
    shape = spec["shape"]
    out, meta = {}, {}
    if name == "c5":
        for t in spec["sampled_t"]:
            vol = syn.series_timestep(shape, t, spec["timesteps"])
            seeds = syn.seeds_streamed(shape, spec["seeds"], t=t, steps=spec["timesteps"])
            top_fixture(vol, seeds, spec, f"t{t}_", out, meta)
    else:
        vol = syn.phantom_streamed(shape)
        seeds = syn.seeds_streamed(shape, spec["seeds"])
        top_fixture(vol, seeds, spec, "", out, meta)
    np.savez_compressed(os.path.join(HERE, f"{name}_top.npz"), **out)
    entry = dict(spec, top=meta, tol=TOP.tol, beta=TOP.beta, min_weight=TOP.min_weight,
                 npz_sha256=hashlib.sha256(open(os.path.join(HERE, f"{name}_top.npz"), "rb").read()).hexdigest())
    path = os.path.join(HERE, "MANIFEST.json")
    with open(path) as f:
        manifest = json.load(f)
    manifest.setdefault("bench", {})[name] = json.loads(json.dumps(entry))
    with open(path, "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or ["c3", "c5", "c4"]:
        make(n)
