"""Where a step goes outside the solve kernels (diagnostics): CUDA events around the phases of
device.hierarchical_random_walker, replayed phase by phase.   python tools/step_timeline.py [c4|c3|c2]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math
import torch
from bench import WORKLOADS, host_inputs
from paper_2509_26213_b200 import device
from paper_2509_26213_b200.config import RWConfig

wl = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
shape, brick, L = tuple(wl["shape"]), tuple(wl["brick"]), wl["levels"]
vh, sh = host_inputs(shape)
vol, sd = vh.cuda(), sh.cuda()
del vh, sh
ws = device.Workspace()
cfg = RWConfig()
for _ in range(2):
    device.hierarchical_random_walker(vol, sd, brick, L, cfg, workspace=ws)
torch.cuda.synchronize()
ev = lambda: torch.cuda.Event(enable_timing=True)
marks = [("start", ev())]
marks[-1][1].record()
vols = device.lod_chain(vol, brick, L)
marks.append(("lod", ev())); marks[-1][1].record()
seeds = [sd]
for _ in range(L - 1):
    seeds.append(device.project_seeds(seeds[-1]))
marks.append(("seeds", ev())); marks[-1][1].record()
top = L - 1
p_top, st_top = device.solve_level(vols[top], seeds[top], tuple(vols[top].shape), None, cfg, workspace=ws)
marks.append(("coarsest", ev())); marks[-1][1].record()
probs = {top: p_top}
cg = {top: st_top["cg_ms"]}
for k in range(top - 1, -1, -1):
    nb = math.prod(device.brick_grid(vols[k].shape, brick))
    chunks = 8 if nb >= 16384 else (2 if nb >= 4096 else 1)
    if chunks > 1:
        lab = torch.empty(vols[k].shape, dtype=torch.uint8, device="cuda") if k == 0 else None
        probs[k], parts = device._solve_level_chunked(vols[k], seeds[k], brick, probs[k + 1], cfg, lab, ws, chunks, None)
        torch.cuda.synchronize()
        cg[k] = sum(device._resolve(p)["cg_ms"] for p in parts)
    else:
        x = device.upsample(probs[k + 1], vols[k].shape)
        probs[k], st = device.solve_level(vols[k], seeds[k], brick, x, cfg, workspace=ws)
        cg[k] = st["cg_ms"]
    marks.append((f"level{k}", ev())); marks[-1][1].record()
torch.cuda.synchronize()
for (a, ea), (b, eb) in zip(marks, marks[1:]):
    lvl = b[5:] if b.startswith("level") else None
    k = int(lvl) if lvl is not None else (top if b == "coarsest" else None)
    extra = f" (solve kernels {cg[k]:.2f} ms)" if k is not None else ""
    print(f"{b:10s} {ea.elapsed_time(eb):7.2f} ms{extra}")
print(f"total      {marks[0][1].elapsed_time(marks[-1][1]):7.2f} ms")
