"""LOD step timing at config 4 sizes (diagnostics): lod_down 1024^3 -> 512^3 -> 256^3 -> 128^3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_26213_b200 import device

vol = torch.rand((1024, 1024, 1024), device="cuda")
for _ in range(2):
    lv = device.lod_chain(vol, (32, 32, 32), 4)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    lv = device.lod_chain(vol, (32, 32, 32), 4)
e1.record()
torch.cuda.synchronize()
print(f"lod_chain 1024^3, 4 levels: {e0.elapsed_time(e1) / 5:.3f} ms per pyramid")
