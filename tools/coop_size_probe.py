import os, sys, torch
sys.path.insert(0, '/root/repo')
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
for n in (64, 128):
    vol = synthetic.phantom_device((n,)*3); sd = synthetic.seeds_device((n,)*3, "S1")
    for _ in range(2):
        prob, st = device.solve_level(vol, sd, (n,)*3, None, RWConfig())
    torch.cuda.synchronize()
    print(n, os.environ.get("RWB_LIBRARY","base").split("/")[-1], round(st["cg_ms"],3), st["iterations_max"])
