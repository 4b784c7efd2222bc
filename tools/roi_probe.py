"""Region-limited hierarchy and the brick-skip rule at config 4 (diagnostics): full solve vs the
lazy solve of viewport-sized regions, and vs skipping decided bricks (bricks per level, device ms)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import host_inputs
from paper_2509_26213_b200 import device
from paper_2509_26213_b200.config import RWConfig

shape = (1024, 1024, 1024)
vh, sh = host_inputs(shape)
vol, sd = vh.cuda(), sh.cuda()
del vh, sh
ws = device.Workspace()
cases = [("full", None), ("roi 256^3 centre", ((384, 384, 384), (640, 640, 640))),
         ("roi 1024x1024x32 slab", ((496, 0, 0), (528, 1024, 1024))), ("roi 64^3 blob A", ((275, 480, 480), (339, 544, 544)))]
cases += [("skip_eps 1e-4", "skip1e-4"), ("skip_eps 1e-3", "skip1e-3")]
full = None
for name, roi in cases:
    cfg = RWConfig()
    if isinstance(roi, str):
        cfg, roi = RWConfig(skip_eps=float(roi[4:])), None
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 4, cfg, workspace=ws, roi=roi)
        e1.record()
        torch.cuda.synchronize()
    extra = ""
    if full is None:
        full = res.prob.clone()
    elif cfg.skip_eps is not None:
        extra = f", skipped {[s.get('skipped') for s in res.stats]}, max |p - p_full| {float((res.prob - full).abs().max()):.2e}"
    print(f"{name}: {e0.elapsed_time(e1):.1f} ms, bricks per level {[s['bricks'] for s in res.stats]}{extra}", flush=True)
