"""Parity at the BENCHMARKED configurations, full size, at the bench's settings (`RWConfig()`:
beta 100, w_min 1e-6, tol 1e-6 — `bench.py` BETA/WMIN/TOL).

Inputs are the §8(d) generator (`synthetic.phantom_streamed` = `default_rng(0xC0FFEE)`, the input
`bench.py` segments).  Per configuration:

1. the GPU pyramid (LOD levels, projected seeds) equals the oracle's bit for bit (SHA-256 frozen by
   `tests/golden/make_bench_fixtures.py`);
2. the coarsest (whole-level) solve matches the oracle's tol-1e-10 solve frozen in the fixture;
3. every finer level: a fixed random sample of bricks (64 per level) is solved by the float64 oracle
   from the GPU's OWN parent level (`oracle.rw.solve_brick`) and compared with the GPU's bricks.

Bars (BASELINE.json north_star): |p_gpu - p_oracle| <= 1e-4; labels equal outside |p - 0.5| <= 1e-4.
"""

import hashlib
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import rw as orw  # noqa: E402
from paper_2509_26213_b200 import api, device, synthetic  # noqa: E402
from paper_2509_26213_b200.config import RWConfig  # noqa: E402

with open(os.path.join(GOLDEN, "MANIFEST.json")) as f:
    BENCH = json.load(f).get("bench", {})

PROB_TOL = 1e-4
BAND = 1e-4
BENCH_CFG = RWConfig()  # the bench's tolerance (1e-6) and parameters
TIGHT = orw.RWParams(tol=1e-10, max_iter=50000)
SAMPLES = 64


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def assert_parity(p_gpu, p_ref, lab_gpu=None, what=""):
    err = float(np.abs(p_gpu.astype(np.float64) - p_ref).max()) if p_ref.size else 0.0
    assert err <= PROB_TOL, f"{what}: max |p_gpu - p_oracle| = {err:.3e} > {PROB_TOL}"
    if lab_gpu is not None:
        band = np.abs(p_ref - 0.5) <= BAND
        bad = (lab_gpu != (p_ref > 0.5)) & ~band
        assert not bad.any(), f"{what}: {int(bad.sum())} label mismatches outside the 0.5 band"
    return err


def check_pyramid(res, meta):
    for k, (v, s) in enumerate(zip(res.volumes, res.seeds)):
        assert sha(host(v)) == meta["volume_sha256"][k], f"LOD level {k} differs from the oracle's"
        assert sha(host(s)) == meta["seeds_sha256"][k], f"seed level {k} differs from the oracle's"


def check_top(res, fixture, stride):
    top = host(res.levels[-1])
    sub = tuple(slice(None, None, stride) for _ in top.shape)
    return assert_parity(top[sub], fixture.astype(np.float64), what="coarsest level")


def check_sampled_bricks(res, brick, seed, n=SAMPLES, labels0=None):
    """Levels top-1 .. 0: `n` random bricks each, oracle-solved from the GPU's parent level."""
    rng = np.random.default_rng(seed)
    worst = {}
    for k in range(len(res.levels) - 2, -1, -1):
        vol = host(res.volumes[k])
        seeds = host(res.seeds[k])
        parent = host(res.levels[k + 1])
        prob = host(res.levels[k])
        grid = [-(-s // b) for s, b in zip(vol.shape, brick)]
        total = int(np.prod(grid))
        picks = rng.choice(total, size=min(n, total), replace=False)
        hs = [np.unravel_index(int(i), grid) for i in picks]

        def one(h):
            box, p_ref, _ = orw.solve_brick(vol, seeds, parent, brick, h, TIGHT)
            return h, box, p_ref

        with ThreadPoolExecutor(max_workers=len(os.sched_getaffinity(0))) as pool:
            results = list(pool.map(one, hs))
        errs = []
        for h, box, p_ref in results:
            lab = labels0[box] if (k == 0 and labels0 is not None) else None
            errs.append(assert_parity(prob[box], p_ref, lab, what=f"level {k} brick {tuple(int(x) for x in h)}"))
        worst[k] = max(errs)
    return worst


def _fixture(name):
    if name not in BENCH:
        pytest.fail(f"tests/golden/MANIFEST.json has no '{name}' bench fixture (make_bench_fixtures.py)")
    return BENCH[name], load_golden(f"{name}_top.npz")


def test_config4_full_size_vs_oracle():
    """Config 4 (1024^3, 4 levels, 32^3 bricks): the benchmarked configuration, brick-resident q4
    engine on levels 0-2, cooperative whole-level solve on the 128^3 coarsest level."""
    spec, fx = _fixture("c4")
    meta = spec["top"]["top"]
    shape, brick = tuple(spec["shape"]), tuple(spec["brick"])
    vol = synthetic.phantom_streamed(shape)
    seeds = synthetic.seeds_streamed(shape, spec["seeds"])
    assert sha(vol) == meta["volume_sha256"][0] and sha(seeds) == meta["seeds_sha256"][0]
    res = device.hierarchical_random_walker(torch.from_numpy(vol).cuda(), torch.from_numpy(seeds).cuda(), brick,
                                            spec["levels"], BENCH_CFG)
    del vol
    assert [s["path"] for s in res.stats] == [1, 1, 1, 3]
    assert all(s["not_converged"] == 0 for s in res.stats)
    check_pyramid(res, meta)
    check_top(res, fx["top_prob"], spec["stride"])
    worst = check_sampled_bricks(res, brick, seed=4, labels0=host(res.labels))
    print("config 4 worst sampled |dp| per level:", worst)


def test_config3_full_size_vs_oracle():
    """Config 3 (16384^2, 9 levels, 64^2 tiles): tile-resident engine on levels 0-7, whole-level
    solve of the 64^2 coarsest level."""
    spec, fx = _fixture("c3")
    meta = spec["top"]["top"]
    shape, brick = tuple(spec["shape"]), tuple(spec["brick"])
    vol = synthetic.phantom_streamed(shape, slab=1024)
    seeds = synthetic.seeds_streamed(shape, spec["seeds"], slab=1024)
    assert sha(vol) == meta["volume_sha256"][0]
    res = device.hierarchical_random_walker(torch.from_numpy(vol).cuda(), torch.from_numpy(seeds).cuda(), brick,
                                            spec["levels"], BENCH_CFG)
    assert all(s["not_converged"] == 0 for s in res.stats)
    assert res.stats[0]["path"] == 1 and res.stats[-1]["path"] == 1  # 64^2 top: one tile-resident CTA
    check_pyramid(res, meta)
    check_top(res, fx["top_prob"], spec["stride"])
    check_sampled_bricks(res, brick, seed=3, labels0=host(res.labels))


def test_config5_series_vs_oracle():
    """Config 5 (512^3 x 16 timesteps, host series streamed through api.segment_series): three
    timesteps of the series checked like config 4 — coarsest level against the fixture, sampled
    bricks of every finer level from the GPU's parent."""
    spec, fx = _fixture("c5")
    shape, brick, steps = tuple(spec["shape"]), tuple(spec["brick"]), spec["timesteps"]
    ts = list(spec["sampled_t"])
    # a 3-timestep series in pinned host memory through the public 4-D entry point
    vol = torch.empty((len(ts),) + shape, dtype=torch.float32).pin_memory()
    sd = torch.empty((len(ts),) + shape, dtype=torch.uint8).pin_memory()
    for i, t in enumerate(ts):
        synthetic.series_timestep(shape, t, steps, out=vol[i].numpy())
        synthetic.seeds_streamed(shape, spec["seeds"], t=t, steps=steps, out=sd[i].numpy())
    prob, labels = api.segment_series(vol, sd, brick, spec["levels"], BENCH_CFG)
    for i, t in enumerate(ts):
        meta = spec["top"][f"t{t}_"]
        assert sha(vol[i].numpy()) == meta["volume_sha256"][0]
        res = device.hierarchical_random_walker(vol[i].cuda(), sd[i].cuda(), brick, spec["levels"], BENCH_CFG)
        # the streamed series result is the per-timestep device result, byte for byte
        np.testing.assert_array_equal(prob[i].numpy(), host(res.prob))
        np.testing.assert_array_equal(labels[i].numpy(), host(res.labels))
        check_pyramid(res, meta)
        check_top(res, fx[f"t{t}_top_prob"], spec["stride"])
        check_sampled_bricks(res, brick, seed=50 + t, n=24, labels0=labels[i].numpy())
