"""PLCT streaming throughput on the box (diagnostics): save a device volume as a chunked file,
drop it from nothing (page cache stays warm), load it back, time both; segment_file end to end."""
import os, sys, time, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_26213_b200 import plct, synthetic
from paper_2509_26213_b200.config import RWConfig

n = int(os.environ.get("PT_N", "512"))
shape, chunk = (n,) * 3, (32, 32, 32)
vol = synthetic.phantom_device(shape); sd = synthetic.seeds_device(shape, "S1")
d = tempfile.mkdtemp(dir=os.environ.get("PT_DIR", "/tmp"))
for rep in range(2):
    t = time.perf_counter(); plct.save(vol, f"{d}/v.plct", chunk); plct.save(sd, f"{d}/s.plct", chunk)
    torch.cuda.synchronize(); ts = time.perf_counter() - t
    t = time.perf_counter(); v2, _ = plct.load(f"{d}/v.plct"); s2, _ = plct.load(f"{d}/s.plct")
    torch.cuda.synchronize(); tl = time.perf_counter() - t
    gb = vol.numel() * 5 / 1e9
    print(f"{n}^3: save {gb / ts:.1f} GB/s ({ts * 1e3:.0f} ms), load {gb / tl:.1f} GB/s ({tl * 1e3:.0f} ms), equal",
          bool(torch.equal(v2, vol) and torch.equal(s2, sd)), flush=True)
t = time.perf_counter()
plct.segment_file(f"{d}/v.plct", f"{d}/s.plct", f"{d}/p.plct", f"{d}/l.plct", levels=4 if n >= 512 else 2, cfg=RWConfig())
torch.cuda.synchronize(); te = time.perf_counter() - t
print(f"segment_file {n}^3 file to file: {te * 1e3:.0f} ms, {vol.numel() / te / 1e9:.2f} G voxel/s")
