"""Phase timeline of the multigrid whole-level solve (RWB_MG_TRACE=1; diagnostics): per iteration,
the %globaltimer stamps of block 0 at the phase boundaries (rwb_mgcg.cu `stamp`)."""
import ctypes, os, sys
os.environ["RWB_MG_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_26213_b200 import _native, device, synthetic
from paper_2509_26213_b200.config import RWConfig

n0, lv = int(sys.argv[1]) if len(sys.argv) > 1 else 256, int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
shape = (n0,) * 3
vol = torch.from_numpy(synthetic.phantom_streamed(shape)).to(dev)
sd = torch.from_numpy(synthetic.seeds_streamed(shape, "S1")).to(dev)
vols = device.lod_chain(vol, (32, 32, 32), lv)
s = sd
for _ in range(lv - 1):
    s = device.project_seeds(s)
top = vols[-1]
for _ in range(2):
    p, st = device.solve_level(top, s, top.shape, None, RWConfig())
torch.cuda.synchronize()
print("iters", st["iterations_max"], "cg_ms", st["cg_ms"])
lib = _native.lib()
buf = (ctypes.c_ulonglong * 128)()
lib.rwb_mg_trace_dump(buf)
t = np.array(buf[:], dtype=np.int64).reshape(8, 16)
names = {0: "start", 1: "down0", 2: "bar", 3: "down-grid", 4: "cta0", 5: "bar", 6: "up-grid", 7: "up0", 8: "bar",
         9: "cg", 10: "bar"}
print("build (ns):", int(t[0, 15] - t[0, 14]), "seg", os.environ.get("RWB_MG_SEG", "16"))
for it in range(1, 6):
    row = t[it]
    d = {names[k]: int(row[k] - row[k - 1]) for k in range(1, 11)}
    d["total"] = int(t[it + 1, 0] - row[0]) if it < 7 else None
    print(it, d)
