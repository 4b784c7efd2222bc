"""Whole-level multigrid solve time on small levels (diagnostics): config 3's 64^2 top and a few
other small whole levels, cg_ms and iterations (RWB_MG_ONE_CTA_CELLS selects the one-CTA path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig

for shape in [(64, 64), (128, 128), (32, 32, 32), (40, 40, 40), (64, 64, 64)]:
    vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
    sd = torch.from_numpy(synthetic.seeds(shape, "S1")).cuda()
    for cfg, tag in [(RWConfig(multigrid=True), "mg"), (RWConfig(multigrid=False), "jacobi")]:
        for _ in range(3):
            p, st = device.solve_level(vol, sd, shape, None, cfg)
        torch.cuda.synchronize()
        print(shape, tag, "iters", st["iterations_max"], "cg_ms %.3f" % st["cg_ms"], flush=True)
