"""Finish-time spread of the resident engine's clusters for one level solve (diagnostics; needs
librwb_trace.so built with -DRWB_TRACE)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2509_26213_b200 import _native
_native.load_library(os.path.join(_native.LIB_DIR, "librwb_trace.so"))
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
lib = _native.load_library()
lib.rwb_end_dump.argtypes = [ctypes.c_void_p]
n = int(os.environ.get("TAIL_N", "512"))
shape = (n,) * 3
vol = synthetic.phantom_device(shape); sd = synthetic.seeds_device(shape, "S1")
res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 2, RWConfig(cluster=8), level0_chunks=1)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 64)()
lib.rwb_end_dump(buf)
t = np.array(buf[:15], dtype=np.float64)
st = res.stats[0]
print("level-0 solve ms", round(st["cg_ms"], 2), "bricks", st["bricks"])
print("cluster finish spread (ms): max-min", round((t.max() - t.min()) / 1e6, 3), "max-median", round((t.max() - np.median(t)) / 1e6, 3))
