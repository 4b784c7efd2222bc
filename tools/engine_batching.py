"""Operator mode through the reference Engine: random-walker hierarchy with per-chunk tasks
(max_requests_per_task=1) against batched tasks (diagnostics for SURVEY 8(f)3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_26213_b200 import ops as rwops, synthetic, _native

cc = rwops._chunkcast()
from chunkcast.engine import Engine, EngineConfig
from chunkcast.store import StoreConfig

n = int(os.environ.get("EB_N", "256"))
shape, chunk = (n,) * 3, (32, 32, 32)
vol = synthetic.phantom(shape)
sd = synthetic.seeds(shape, "S1")
for per in [int(x) for x in os.environ.get("EB_PER", "1,8,64").split(",")]:
    pyr = rwops.hierarchical_random_walker(cc.ops.source_from_array(vol, chunk), cc.ops.source_from_array(sd, chunk),
                                           levels=2)
    with Engine(EngineConfig(stores=StoreConfig(ram_capacity=8 << 30), worker_pool_size=int(os.environ.get("EB_WORKERS", "8")),
                             max_requests_per_task=per)) as eng:
        t0 = time.perf_counter()
        positions = list(pyr.node(0).md.chunk_positions())
        eng.resolve(pyr.node(0), positions)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{n}^3, max_requests_per_task={per}: {dt * 1e3:.0f} ms, {vol.size / dt / 1e6:.1f} M voxel/s", flush=True)
