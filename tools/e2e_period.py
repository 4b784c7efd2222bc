"""Steady-state period of api.segment_many at config 4 (diagnostics): times K1 and K2 volumes through
the streaming API and reports (t(K2) - t(K1)) / (K2 - K1), plus the allocator's activity.

    python tools/e2e_period.py [K1] [K2] [level0_chunks]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__ as entry  # noqa: E402

entry.build()
from bench import host_inputs  # noqa: E402
from paper_2509_26213_b200 import api, device  # noqa: E402
from paper_2509_26213_b200.config import RWConfig  # noqa: E402

K1 = int(sys.argv[1]) if len(sys.argv) > 1 else 3
K2 = int(sys.argv[2]) if len(sys.argv) > 2 else 7
chunks = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "auto" else None
shape = (1024,) * 3
vol_h, seeds_h = host_inputs(shape)
outs = [(torch.empty(shape, dtype=torch.float32, pin_memory=True), torch.empty(shape, dtype=torch.uint8, pin_memory=True))
        for _ in range(2)]
ws = device.Workspace()
cfg = RWConfig()


def run(k):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = torch.cuda.current_stream()
    h0 = time.perf_counter()
    e0.record(s)
    api.segment_many([(vol_h, seeds_h)] * k, (32, 32, 32), 4, cfg, outputs=outs, workspace=ws, cyclic_outputs=True,
                     level0_chunks=chunks)
    e1.record(s)
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), (h1 - h0) * 1e3


run(2)
st0 = torch.cuda.memory_stats()
t1, h1 = run(K1)
t2, h2 = run(K2)
st1 = torch.cuda.memory_stats()
print(f"K={K1}: {t1:.1f} ms ({t1 / K1:.1f}/vol, host enqueue {h1:.0f} ms); K={K2}: {t2:.1f} ms ({t2 / K2:.1f}/vol, "
      f"host enqueue {h2:.0f} ms); steady-state period {(t2 - t1) / (K2 - K1):.1f} ms")
for key in ("num_alloc_retries", "num_device_alloc", "num_device_free", "num_sync_all_streams"):
    print(key, st1.get(key, 0) - st0.get(key, 0))
print("reserved GB", torch.cuda.memory_reserved() / 1e9)
