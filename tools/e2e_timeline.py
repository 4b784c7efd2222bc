"""Per-stream timeline of api.segment_many at the bench shape (diagnostics)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_26213_b200 import api, device, synthetic
from paper_2509_26213_b200.config import RWConfig

n = int(os.environ.get("TL_N", "1024"))
shape = (n,) * 3
vol = synthetic.phantom_device(shape).cpu().pin_memory()
sd = synthetic.seeds_device(shape).cpu().pin_memory()
outs = [(torch.empty(shape, dtype=torch.float32, pin_memory=True), torch.empty(shape, dtype=torch.uint8, pin_memory=True))
        for _ in range(2)]
ws = device.Workspace()
cfg = RWConfig()
api.segment_many([(vol, sd)] * 2, (32, 32, 32), 4, cfg, outputs=outs, workspace=ws)
torch.cuda.synchronize()

# monkeypatch Event.record to log (stream, tag, event)
log = []
orig_hrw = device.hierarchical_random_walker


import time
T0 = [0.0]


def hrw(*a, **k):
    print(f"host: compute submit at {(time.perf_counter() - T0[0]) * 1e3:8.1f} ms", flush=True)
    s = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True); e0.record(s)
    r = orig_hrw(*a, **k)
    e1 = torch.cuda.Event(enable_timing=True); e1.record(s)
    log.append(("compute", e0, e1))
    return r


device.hierarchical_random_walker = hrw
orig_copy = torch.Tensor.copy_


def copy_(self, src, non_blocking=False):
    s = torch.cuda.current_stream()
    e0 = torch.cuda.Event(enable_timing=True); e0.record(s)
    r = orig_copy(self, src, non_blocking)
    e1 = torch.cuda.Event(enable_timing=True); e1.record(s)
    tag = "h2d" if self.is_cuda else "d2h"
    log.append((tag, e0, e1))
    return r


torch.Tensor.copy_ = copy_
base = torch.cuda.Event(enable_timing=True)
base.record()
torch.cuda.synchronize()
T0[0] = time.perf_counter()
print(torch.cuda.memory_allocated() / 1e9, torch.cuda.memory_reserved() / 1e9, flush=True)
api.segment_many([(vol, sd)] * 5, (32, 32, 32), 4, cfg, outputs=outs, workspace=ws)
torch.cuda.synchronize()
torch.Tensor.copy_ = orig_copy
print(torch.cuda.memory_allocated() / 1e9, torch.cuda.memory_reserved() / 1e9, torch.cuda.memory_stats().get("num_alloc_retries"), flush=True)
for tag, e0, e1 in log:
    print(f"{tag:8s} {base.elapsed_time(e0):8.1f} -> {base.elapsed_time(e1):8.1f}  ({e0.elapsed_time(e1):6.1f} ms)")
