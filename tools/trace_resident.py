"""Phase timing of the brick-resident CG loop (diagnostics; needs librwb_trace.so built with -DRWB_TRACE)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2509_26213_b200 import _native
_native.load_library(os.path.join(_native.LIB_DIR, "librwb_trace.so"))
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
shape = (256, 256, 256)
vol = synthetic.phantom_device(shape); sd = synthetic.seeds_device(shape, "S1")
res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 2, RWConfig(cluster=8), level0_chunks=1)
torch.cuda.synchronize()
print(res.stats[0])
buf = (ctypes.c_longlong * (8 * 64 * 8))()
lib = _native.load_library()
lib.rwb_trace_dump.argtypes = [ctypes.c_void_p]
print("rc", lib.rwb_trace_dump(buf))
t = np.frombuffer(buf, dtype=np.int64).reshape(8, 64, 8)
names = ["spmv", "warp_sums+push", "wait", "scalars", "update+publish", "-"]
ncol = 7
for rank in (0, 3, 7):
    d = np.diff(t[rank][:, :ncol], axis=1)[5:40]
    tot = (t[rank, 6:41, 0] - t[rank, 5:40, 0])
    print("rank", rank, "median cycles per phase", dict(zip(names, np.median(d, axis=0).astype(int))), "iter", int(np.median(tot)))
st = t[:, 5:40, 0]
print("start skew (max-min) median", int(np.median(st.max(0) - st.min(0))))

bbuf = (ctypes.c_longlong * (8 * 16 * 10))()
lib.rwb_btrace_dump.argtypes = [ctypes.c_void_p]
lib.rwb_btrace_dump(bbuf)
b = np.frombuffer(bbuf, dtype=np.int64).reshape(8, 16, 10)
bn = ["staging_wait", "registers", "iterations", "(0)", "(0)", "(0)", "writeback", "(0)"]
for rank in (0, 7):
    cols = [0, 1, 2, 6, 7]
    d = np.diff(b[rank, 1:12][:, cols], axis=1)
    bn2 = ["staging_wait", "registers", "iterations", "writeback"]
    print("rank", rank, "median cycles per brick phase", dict(zip(bn2, np.median(d, axis=0).astype(int))),
          "brick", int(np.median(b[rank, 2:12, 0] - b[rank, 1:11, 0])))
