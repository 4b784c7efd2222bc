"""Short, ncu-friendly runs of the dominant kernels at bench shapes.

    python tools/ncu_target.py streaming [--config c4] [--level 0] [--iters 4]
        CG iterations of one level with direct (non-graph) launches, all bricks active,
        so `ncu -k regex:cg_pass` sees ordinary kernel launches of bench shapes.
    python tools/ncu_target.py hierarchy [--config c4] [--levels N]
        one full hierarchical solve of the bench inputs (multigrid coarsest level, then
        brick-resident levels): at C4 `ncu -k regex:resident3d_q4 -s 3 -c 1` captures the first
        level-0 slab (launch order: level 2 x1, level 1 x2, level 0 x8).
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import __graft_entry__ as entry  # noqa: E402

entry.build()
from bench import WORKLOADS  # noqa: E402
from paper_2509_26213_b200 import device, synthetic  # noqa: E402
from paper_2509_26213_b200.config import RWConfig  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("mode", choices=["streaming", "hierarchy"])
ap.add_argument("--config", default="c4")
ap.add_argument("--level", type=int, default=0)
ap.add_argument("--iters", type=int, default=4)
args = ap.parse_args()
wl = WORKLOADS[args.config]
if args.mode == "hierarchy":  # the bench's inputs (SURVEY.md 8(d) numpy generator)
    from bench import host_inputs

    vh, sh = host_inputs(wl["shape"])
    vol, seeds = vh.cuda(), sh.cuda()
    del vh, sh
else:
    vol = synthetic.phantom_device(wl["shape"])
    seeds = synthetic.seeds_device(wl["shape"], "S1")
if args.mode == "hierarchy":
    res = device.hierarchical_random_walker(vol, seeds, wl["brick"], wl["levels"], RWConfig())
    torch.cuda.synchronize()
    print(res.stats)
    sys.exit(0)
vols = device.lod_chain(vol, wl["brick"], wl["levels"])
sl = [seeds]
for _ in range(len(vols) - 1):
    sl.append(device.project_seeds(sl[-1]))
k = args.level
top = len(vols) - 1
if k == top:
    brick, bound = tuple(vols[k].shape), None
else:
    brick = wl["brick"]
    parent = torch.full(vols[k + 1].shape, 0.5, device="cuda")
    bound = device.upsample(parent, vols[k].shape)
cfg = RWConfig(tol=1e-30, max_iter=args.iters, check_every=2, use_graph=False, resident=False)
out, st = device.solve_level(vols[k], sl[k], brick, bound, cfg)
torch.cuda.synchronize()
print(st)
