import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
for shape, chunk, levels in [((64, 64, 64), (32, 32, 32), 2), ((40, 36, 28), (16, 16, 16), 2), ((96, 80), (32, 32), 3)]:
    vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
    sd = torch.from_numpy(synthetic.seeds(shape, "S1")).cuda()
    res = device.hierarchical_random_walker(vol, sd, chunk, levels, RWConfig(tol=1e-7))
    torch.cuda.synchronize()
    print(shape, "ok", float(res.prob.mean()))
    for k in range(1, levels):
        fine = res.volumes[k - 1].shape
        out = device.upsample(res.levels[k], fine)
        torch.cuda.synchronize()
        print("  upsample", tuple(res.levels[k].shape), "->", tuple(fine), "ok")
