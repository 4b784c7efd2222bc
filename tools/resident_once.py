"""One 256^3, 2-level hierarchical solve with a chosen resident-engine variant (ncu target).

    python tools/resident_once.py [cluster]      # ncu -k regex:resident3d -c 1 ...
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
cl = int(sys.argv[1]) if len(sys.argv) > 1 else 8
shape = (256, 256, 256)
vol = synthetic.phantom_device(shape); sd = synthetic.seeds_device(shape, "S1")
res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 2, RWConfig(cluster=cl), level0_chunks=1)
torch.cuda.synchronize()
print(res.stats[0]["cg_ms"])
