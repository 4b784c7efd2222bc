"""Step time of a hierarchy for several level-0 slab counts (diagnostics).

    python tools/cmp_chunks.py c4 1 4 8
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import WORKLOADS
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig

wl = WORKLOADS[sys.argv[1]]
vol = synthetic.phantom_device(wl["shape"]); sd = synthetic.seeds_device(wl["shape"])
ws = device.Workspace()
for rep in range(2):
    for c in [int(x) for x in sys.argv[2:]]:
        res = device.hierarchical_random_walker(vol, sd, wl["brick"], wl["levels"], RWConfig(), workspace=ws, level0_chunks=c)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = device.hierarchical_random_walker(vol, sd, wl["brick"], wl["levels"], RWConfig(), workspace=ws, level0_chunks=c)
        e1.record()
        torch.cuda.synchronize()
        print(sys.argv[1], "chunks", c, round(e0.elapsed_time(e1), 2), "L0 solve ms", round(res.stats[0]["cg_ms"], 2))
