"""Which library call makes the next work on the compute stream wait for a D2H on another stream? (diagnostics)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig

n = 4 << 30
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
comp = torch.cuda.Stream()
down = torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)
shape = (128, 128, 128)
vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
sd = torch.from_numpy(synthetic.seeds(shape, "S1")).cuda()
ws = device.Workspace()


def work(kind):
    if kind == "sleep":
        torch.cuda._sleep(20_000_000)
    elif kind == "lod":
        device.lod_chain(vol, (32, 32, 32), 3)
    elif kind == "solve_resident":
        device.solve_level(vol, sd, (32, 32, 32), torch.rand(shape, device="cuda"), RWConfig(), workspace=ws)
    elif kind == "solve_coop":
        device.solve_level(vol[:64, :64, :64].contiguous(), sd[:64, :64, :64].contiguous(), (64, 64, 64), None,
                           RWConfig(), workspace=ws)
    elif kind == "hrw":
        device.hierarchical_random_walker(vol, sd, (32, 32, 32), 3, RWConfig(), workspace=ws)


for kind in ["sleep", "lod", "solve_resident", "solve_coop", "hrw", "sleep"]:
    with torch.cuda.stream(comp):
        work(kind)
    torch.cuda.synchronize()
    base, c0, c1, m = E(), E(), E(), E()
    base.record(comp)
    with torch.cuda.stream(comp):
        work(kind)
    ev = torch.cuda.Event()
    ev.record(comp)
    with torch.cuda.stream(down):
        down.wait_event(ev)
        c0.record(down)
        h.copy_(d, non_blocking=True)
        c1.record(down)
    m.record(comp)
    torch.cuda.synchronize()
    f = base.elapsed_time
    print(f"{kind:15s} copy {f(c0):7.1f}-{f(c1):7.1f}   next mark on comp at {f(m):7.1f}", flush=True)
