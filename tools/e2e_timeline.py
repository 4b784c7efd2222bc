"""segment_many with events around every step of its loop (diagnostics)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import glob
import numpy as np
import torch
from paper_2509_26213_b200 import api, device, synthetic
from paper_2509_26213_b200.config import RWConfig

n = 1024
shape = (n,) * 3
vol = synthetic.phantom_device(shape).cpu().pin_memory()
sd = synthetic.seeds_device(shape).cpu().pin_memory()
outs = [(torch.empty(shape, dtype=torch.float32, pin_memory=True), torch.empty(shape, dtype=torch.uint8, pin_memory=True))
        for _ in range(2)]
ws = device.Workspace()
_cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*")) + \
    glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*")) + \
    ["/usr/local/cuda/lib64/libcudart.so"]
cudart = ctypes.CDLL(_cands[0])
print("cudart", _cands[0])
cfg = RWConfig()
api.segment_many([(vol, sd)] * 2, (32, 32, 32), 4, cfg, outputs=outs, workspace=ws)
torch.cuda.synchronize()
E = lambda: torch.cuda.Event(enable_timing=True)
marks = []


def mark(tag, s):
    e = E(); e.record(s); marks.append((tag, e))


dev = torch.device("cuda", 0)
comp = torch.cuda.Stream(dev) if os.environ.get("OWN_COMP") else torch.cuda.current_stream(dev)
up = torch.cuda.Stream(dev)
down = torch.cuda.Stream(dev)
vol_d = [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(2)]
sd_d = [torch.empty(shape, dtype=torch.uint8, device=dev) for _ in range(2)]
computed = []
base = E(); base.record(comp)
torch.cuda.synchronize()


def upload(i):
    b = i % 2
    with torch.cuda.stream(up):
        if i >= 2:
            up.wait_event(computed[i - 2])
        mark(f"up{i}.start", up)
        vol_d[b].copy_(vol, non_blocking=True)
        sd_d[b].copy_(sd, non_blocking=True)
        mark(f"up{i}.end", up)
        ev = torch.cuda.Event(); ev.record(up)
    return ev


uploaded = [upload(0)]
N = 4
for i in range(N):
    if i + 1 < N:
        h0 = time.perf_counter()
        uploaded.append(upload(i + 1))
        print(f"host upload({i+1}) call took {(time.perf_counter() - h0) * 1e3:.1f} ms", flush=True)
    mark(f"c{i}.before_wait", comp)
    comp.wait_event(uploaded[i])
    mark(f"c{i}.after_wait", comp)
    with torch.cuda.stream(comp):
        res = device.hierarchical_random_walker(vol_d[i % 2], sd_d[i % 2], (32, 32, 32), 4, cfg, workspace=ws)
    mark(f"c{i}.end", comp)
    ev = torch.cuda.Event(); ev.record(comp); computed.append(ev)
    out_p, out_l = outs[i % 2]
    h0 = time.perf_counter()
    with torch.cuda.stream(down):
        down.wait_event(ev)
        mark(f"dn{i}.start", down)
        if os.environ.get("RAW_D2H"):
            for dst, src in ((out_p, res.prob), (out_l, res.labels)):
                rc = cudart.cudaMemcpyAsync(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.data_ptr()),
                                            ctypes.c_size_t(src.numel() * src.element_size()), 2,
                                            ctypes.c_void_p(down.cuda_stream))
                assert rc == 0, rc
        else:
            out_p.copy_(res.prob, non_blocking=True)
            out_l.copy_(res.labels, non_blocking=True)
        mark(f"dn{i}.end", down)
        res.prob.record_stream(down)
        res.labels.record_stream(down)
    print(f"host d2h({i}) submit took {(time.perf_counter() - h0) * 1e3:.1f} ms", flush=True)
torch.cuda.synchronize()
for tag, e in sorted(marks, key=lambda m: base.elapsed_time(m[1])):
    print(f"{base.elapsed_time(e):8.1f} {tag}")
