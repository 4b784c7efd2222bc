"""Time the C4 hierarchy with resident-solver variants (diagnostics).

usage: python tools/cmp_variants.py [name=RWConfig-kwargs-as-json ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2509_26213_b200 import device, synthetic  # noqa: E402
from paper_2509_26213_b200.config import RWConfig  # noqa: E402

variants = [a.split("=", 1) for a in sys.argv[1:]] or [["cg", "{}"]]
n = int(os.environ.get("CMP_N", "1024"))
vol = synthetic.phantom_device((n,) * 3)
sd = synthetic.seeds_device((n,) * 3)
ws = device.Workspace()
for rep in range(2):
    for name, kw in variants:
        cfg = RWConfig(**json.loads(kw))
        res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 4, cfg, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 4, cfg, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        print(name, round(e0.elapsed_time(e1), 2),
              [(s["path"], round(s["cg_ms"], 2), s["iterations_max"], s["iterations_sum"]) for s in res.stats],
              flush=True)
