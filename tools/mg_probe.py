"""Whole-level (coarsest) solver probe: multigrid-preconditioned CG vs Jacobi-PCG on the 128^3
coarsest levels of configs 2 and 4 (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig

dev = torch.device("cuda", 0)
for name, n0, lv in [("c2", 256, 2), ("c4", 1024, 4)]:
    shape = (n0,) * 3
    vol = torch.from_numpy(synthetic.phantom_streamed(shape)).to(dev)
    sd = torch.from_numpy(synthetic.seeds_streamed(shape, "S1")).to(dev)
    vols = device.lod_chain(vol, (32, 32, 32), lv)
    s = sd
    for _ in range(lv - 1):
        s = device.project_seeds(s)
    top, stop = vols[-1], s
    del vol, sd, vols
    res = {}
    for tag, cfg in [("mg", RWConfig()), ("jacobi", RWConfig(multigrid=False))]:
        for rep in range(3):
            p, st = device.solve_level(top, stop, top.shape, None, cfg)
        torch.cuda.synchronize()
        res[tag] = p.cpu().numpy()
        print(name, tag, "iters", st["iterations_max"], "cg_ms %.3f" % st["cg_ms"], "path", st["path"],
              "us/iter %.2f" % (1e3 * st["cg_ms"] / max(1, st["iterations_max"])), flush=True)
    print(name, "max |mg - jacobi|", float(np.abs(res["mg"] - res["jacobi"]).max()), flush=True)
