"""Per-iteration time and HBM rate of the streaming CG passes (diagnostics): config 4's level 0 (or
--config/--level), all bricks active (tol 1e-30), K1 and K2 iterations, the difference per iteration.
Algorithmic bytes per unknown-iteration: 52 (3-D) / 48 (2-D), rwb_solve.cu header.

    python tools/streaming_probe.py [--config c4] [--level 0] [--k1 4] [--k2 12]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import __graft_entry__ as entry  # noqa: E402

entry.build()
from bench import WORKLOADS, load_peak  # noqa: E402
from paper_2509_26213_b200 import device, synthetic  # noqa: E402
from paper_2509_26213_b200.config import RWConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--level", type=int, default=0)
ap.add_argument("--k1", type=int, default=4)
ap.add_argument("--k2", type=int, default=12)
args = ap.parse_args()
wl = WORKLOADS[args.config]
vol = synthetic.phantom_device(wl["shape"])
seeds = synthetic.seeds_device(wl["shape"], "S1")
vols = device.lod_chain(vol, wl["brick"], wl["levels"])
sl = [seeds]
for _ in range(len(vols) - 1):
    sl.append(device.project_seeds(sl[-1]))
k = args.level
parent = torch.full(vols[k + 1].shape, 0.5, device="cuda")
bound = device.upsample(parent, vols[k].shape)
del vol
ws = device.Workspace()


def run(iters):
    cfg = RWConfig(tol=1e-30, max_iter=iters, check_every=iters, resident=False)
    device.solve_level(vols[k], sl[k], wl["brick"], bound, cfg, workspace=ws)  # warm (graph capture)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out, st = device.solve_level(vols[k], sl[k], wl["brick"], bound, cfg, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), st


t1, s1 = run(args.k1)
t2, s2 = run(args.k2)
per = (t2 - t1) / (args.k2 - args.k1)
unk = s2["unknowns"]
bpu = 52 if len(wl["shape"]) == 3 else 48
peak, src = load_peak()
gbs = bpu * unk / (per / 1e3) / 1e9
print(f"level {k} {tuple(vols[k].shape)} unknowns {unk}: {t1:.2f} ms @{args.k1}, {t2:.2f} ms @{args.k2} -> "
      f"{per:.3f} ms per iteration, {gbs:.0f} GB/s = {gbs / peak:.1%} of {peak:.0f} ({src}); path {s2['path']}")
