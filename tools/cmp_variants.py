"""Time the C4 hierarchy with each resident-solver variant (diagnostics)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__ as e
e.build()
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
vol = synthetic.phantom_device((1024,) * 3); sd = synthetic.seeds_device((1024,) * 3)
ws = device.Workspace()
for cl in (8, 512, 16, 8, 512):
    cfg = RWConfig(cluster=cl)
    res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 4, cfg, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 4, cfg, workspace=ws)
    e1.record(); torch.cuda.synchronize()
    print(cl, round(e0.elapsed_time(e1), 2), [(s["path"], round(s["cg_ms"], 2), s["iterations_sum"]) for s in res.stats])
