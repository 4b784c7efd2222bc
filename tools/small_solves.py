"""Small solves of every engine (diagnostics; run with RWB_DEBUG_SYNC=1 to synchronise after every launch): brick-resident (coarse-corrected
and Jacobi), multigrid whole levels (3-D, ragged, 2-D), the 2-D tile engine on a whole 64^2 level,
the streaming solver, a 2-level hierarchy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig

rng = np.random.default_rng(3)
c = lambda a: torch.from_numpy(a).cuda()
for shape in [(64, 64, 64), (70, 41, 33), (64, 64), (97, 130)]:
    vol, sd = synthetic.phantom(shape), synthetic.seeds(shape, "S1")
    device.solve_level(c(vol), c(sd), shape, None, RWConfig(multigrid=True))
    device.solve_level(c(vol), c(sd), shape, None, RWConfig(multigrid=False))
for shape, brick in [((64, 64, 96), (32, 32, 32)), ((70, 40, 48), (32, 32, 32)), ((130, 201), (64, 64))]:
    vol, sd = synthetic.phantom(shape), synthetic.seeds(shape, "S2")
    bound = c(rng.random(shape).astype(np.float32))
    for cfg in (RWConfig(), RWConfig(coarse=False), RWConfig(resident=False)):
        device.solve_level(c(vol), c(sd), brick, bound, cfg)
vol, sd = synthetic.phantom((128, 96, 64)), synthetic.seeds((128, 96, 64), "S1")
device.hierarchical_random_walker(c(vol), c(sd), (32, 32, 32), 2, RWConfig())
torch.cuda.synchronize()
print("sanitize_small: done")
