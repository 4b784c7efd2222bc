"""Run one fused-setup solve (diagnostics: use under compute-sanitizer)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
shape = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "20,18,16").split(","))
brick = tuple(int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "20,18,16").split(","))
vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
sd = torch.from_numpy(synthetic.seeds(shape, "S1")).cuda()
bound = None if brick == shape else torch.rand(shape, device="cuda")
out, st = device.solve_level(vol, sd, brick, bound, RWConfig(tol=1e-7))
torch.cuda.synchronize()
print(st)
