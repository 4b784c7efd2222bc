"""Phase timing of the 4-CTA brick-resident CG loop (diagnostics; needs librwb_trace.so, tools/build_trace.sh)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2509_26213_b200 import _native
_native.load_library(os.path.join(_native.LIB_DIR, os.environ.get("RWB_TRACE_LIB", "librwb_trace.so")))
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
shape = (256, 256, 256)
vol = synthetic.phantom_device(shape); sd = synthetic.seeds_device(shape, "S1")
res = device.hierarchical_random_walker(vol, sd, (32, 32, 32), 2, RWConfig(cluster=4), level0_chunks=1)
torch.cuda.synchronize()
print(res.stats[0])
buf = (ctypes.c_longlong * (4 * 64 * 8))()
lib = _native.load_library()
lib.rwb_q4_trace_dump.argtypes = [ctypes.c_void_p]
print("rc", lib.rwb_q4_trace_dump(buf))
t = np.frombuffer(buf, dtype=np.int64).reshape(4, 64, 8)
names = ["spmv", "warp_sums+push", "wait", "scalars", "update+publish", "syncthreads"]
for rank in range(4):
    d = np.diff(t[rank][:, :7], axis=1)[5:40]
    tot = (t[rank, 6:41, 0] - t[rank, 5:40, 0])
    print("rank", rank, "median cycles per phase", dict(zip(names, np.median(d, axis=0).astype(int))), "iter", int(np.median(tot)))

# per brick of cluster 0 (CTA rank 0): staging wait, prologue (TMEM weights, coarse setup, initial
# exchange), iterations, epilogue — cycles
pro = (ctypes.c_longlong * (4 * 64 * 8))()
lib.rwb_q4_pro_dump.argtypes = [ctypes.c_void_p]
lib.rwb_q4_pro_dump(pro)
p = np.frombuffer(pro, dtype=np.int64).reshape(4, 64, 8)[0]
ok = p[:, 0] > 0
p = p[ok][2:40]
print("per brick median cycles: staging wait", int(np.median(p[:, 1] - p[:, 0])), "prologue",
      int(np.median(p[:, 2] - p[:, 1])), "iterations+epilogue", int(np.median(p[:, 3] - p[:, 2])),
      "next brick gap", int(np.median(p[1:, 0] - p[:-1, 3])))
print("prologue split: TMEM / registers loaded", int(np.median(p[:, 4] - p[:, 1])), "exchange pushed",
      int(np.median(p[:, 5] - p[:, 4])), "exchange wait", int(np.median(p[:, 6] - p[:, 5])),
      "coarse init + barrier", int(np.median(p[:, 2] - p[:, 6])))
print("epilogue", int(np.median(p[:, 3] - p[:, 7])))
