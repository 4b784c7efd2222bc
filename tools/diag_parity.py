"""Per-level GPU-vs-oracle error for a hierarchical case (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__ as e
e.build()
from oracle import rw as orw
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig

shape = tuple(int(x) for x in sys.argv[1].split("x")) if len(sys.argv) > 1 else (96, 96, 96)
brick = (32,) * len(shape)
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 2
vol = synthetic.phantom(shape); sd = synthetic.seeds(shape, "S1")
ref = orw.hierarchical_random_walker(vol, sd, brick, levels, orw.RWParams(tol=1e-10, max_iter=50000))
for tol in (1e-6, 1e-7, 1e-8):
    for resident in (True, False):
        cfg = RWConfig(tol=tol, max_iter=20000, resident=resident)
        res = device.hierarchical_random_walker(torch.from_numpy(vol).cuda(), torch.from_numpy(sd).cuda(), brick, levels, cfg)
        torch.cuda.synchronize()
        errs = [float(np.abs(p.cpu().numpy() - r).max()) for p, r in zip(res.levels, ref.prob)]
        its = [s["iterations_max"] for s in res.stats]
        print(f"tol={tol:g} resident={resident}: per-level max err {['%.2e' % x for x in errs]} iters {its}")
# coarse level alone with the oracle's own parent: isolate the fine-level solve
top = ref.prob[-1]
for resident in (True, False):
    bound = orw.upsample_linear(top, ref.volumes[0].shape).astype(np.float32)
    want = orw.solve_level(ref.volumes[0], ref.seeds[0], brick, bound.astype(np.float64), orw.RWParams(tol=1e-10)).prob
    out, st = device.solve_level(torch.from_numpy(ref.volumes[0]).cuda(), torch.from_numpy(ref.seeds[0]).cuda(), brick,
                                 torch.from_numpy(bound).cuda(), RWConfig(tol=1e-7, resident=resident))
    print("fine level from exact parent, resident", resident, "err %.2e" % np.abs(out.cpu().numpy() - want).max(), st["iterations_max"])
