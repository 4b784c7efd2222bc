"""Stress the whole-level upsampling kernel over many shapes (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_26213_b200 import device
from oracle import rw as orw
rng = np.random.default_rng(1)
bad = 0
for it in range(300):
    nd = 2 if it % 2 else 3
    fine = tuple(int(x) for x in rng.integers(1, 40, size=nd))
    fine = fine[:-1] + (4 * int(rng.integers(1, 20)),)
    parent = rng.random(device.coarse_shape(fine), dtype=np.float32)
    out = device.upsample(torch.from_numpy(parent).cuda(), fine)
    torch.cuda.synchronize()
    ref = orw.upsample_linear(parent, fine)
    err = np.abs(out.cpu().numpy() - ref).max()
    if err > 2e-7:
        bad += 1
        print("mismatch", fine, err)
print("done, bad =", bad)
