"""Randomised parity sweep of the device hierarchy against the float64 oracle (diagnostics):
ragged 3-D shapes with 32^3 bricks (brick-resident TMEM engine + cooperative coarsest level) and
2-D shapes with 64^2 tiles, random seeds sets, 1-3 levels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import rw as orw
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig

rng = np.random.default_rng(int(os.environ.get("SEED", "7")))
worst = 0.0
for case in range(int(os.environ.get("CASES", "12"))):
    if case % 3 == 2:
        shape = tuple(int(rng.integers(70, 200)) for _ in range(2)); brick = (64, 64)
    else:
        shape = tuple(int(rng.integers(33, 100)) for _ in range(3)); brick = (32, 32, 32)
    levels = int(rng.integers(1, 3))
    vol = synthetic.phantom(shape) + 0.05 * rng.standard_normal(shape).astype(np.float32)
    vol = np.clip(vol, 0, 1).astype(np.float32)
    seeds = synthetic.seeds(shape, "S1" if case % 2 else "S2")
    try:
        res = device.hierarchical_random_walker(torch.from_numpy(vol).cuda(), torch.from_numpy(seeds).cuda(), brick,
                                                levels, RWConfig(tol=1e-7))
    except ValueError as e:  # levels outside the valid range for this shape
        print(case, shape, levels, "skip:", e); continue
    ref = orw.hierarchical_random_walker(vol, seeds, brick, levels, orw.RWParams(tol=1e-10), threads=8)
    err = float(np.abs(res.prob.cpu().numpy() - ref.prob[0]).max())
    band = np.abs(ref.prob[0] - 0.5) <= 1e-4
    mism = int(((res.labels.cpu().numpy() != ref.labels) & ~band).sum())
    worst = max(worst, err)
    print(case, shape, brick, levels, f"max err {err:.2e}", "label mismatches", mism, [s["path"] for s in res.stats], flush=True)
    # brick-wise finest levels are small, well-conditioned systems (1e-4 against the tight oracle);
    # a whole-level fp32 solve at tol 1e-7 is as close as its conditioning allows (labels must match)
    # (path 2 Jacobi-PCG or 3 multigrid-PCG: tools/stop_rule_probe.py shows both stop at the same
    # error in float64 as well, an unseeded pocket the ||r|| <= tol ||b|| rule cannot see)
    whole = res.stats[0]["path"] in (2, 3)
    assert (whole or err < 1e-4) and mism == 0, (case, shape, err, mism)
print("worst", worst)
