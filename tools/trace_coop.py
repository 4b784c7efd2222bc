"""Phase timing of the cooperative whole-level CG (diagnostics; librwb_trace.so, tools/build_trace.sh)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2509_26213_b200 import _native
_native.load_library(os.path.join(_native.LIB_DIR, "librwb_trace.so"))
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig
n = int(os.environ.get("COOP_N", "128"))
vol = synthetic.phantom_device((n,) * 3); sd = synthetic.seeds_device((n,) * 3, "S1")
for _ in range(2):
    prob, st = device.solve_level(vol, sd, (n,) * 3, None, RWConfig())
torch.cuda.synchronize()
print(st)
buf = (ctypes.c_longlong * (2 * 64 * 8))()
lib = _native.load_library()
lib.rwb_coop_trace_dump.argtypes = [ctypes.c_void_p]
lib.rwb_coop_trace_dump(buf)
t = np.frombuffer(buf, dtype=np.int64).reshape(2, 64, 8)
names = ["pass1+blocksum", "sync1", "total1", "pass2+blocksum", "sync2", "total2"]
for b in range(2):
    d = np.diff(t[b][:, :7], axis=1)[10:60]
    it = t[b, 11:61, 0] - t[b, 10:60, 0]
    print("block", ["first", "last"][b], dict(zip(names, np.median(d, axis=0).astype(int))), "iter", int(np.median(it)))
