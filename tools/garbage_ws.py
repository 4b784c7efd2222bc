"""Single-threaded solves on workspace memory pre-filled with garbage (diagnostics: does any
kernel read scratch it did not write?)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_26213_b200 import device, synthetic
from paper_2509_26213_b200.config import RWConfig

vol_full = torch.from_numpy(synthetic.phantom((96, 96, 96))).cuda()
sd_full = torch.from_numpy(synthetic.seeds((96, 96, 96), "S1")).cuda()
for fill in (0xFF, 0x7F, 0x00, 0x80):
    for it in range(20):
        z0 = 32 * (it % 3)
        lo = [max(z0 - 1, 0), 31, 31]
        hi = [min(z0 + 33, 96), 65, 65]
        vol = vol_full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].contiguous()
        sd = sd_full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].contiguous()
        bound = torch.rand(vol.shape, device="cuda")
        origin = tuple(-(a % 32) for a in lo)
        grid = device.brick_grid(vol.shape, (32, 32, 32), origin)
        idx = 0
        for hd, a, gdim in zip([z0 // 32, 1, 1], lo, grid):
            idx = idx * gdim + (hd - a // 32)
        bl = torch.tensor([idx], dtype=torch.int32, device="cuda")
        nbytes = device.workspace_bytes(vol.shape, (32, 32, 32), 1, origin)
        ws = device.Workspace()
        ws.buffer = torch.full((nbytes,), fill, dtype=torch.uint8, device="cuda")
        prob, st = device.solve_level(vol, sd, (32, 32, 32), bound, RWConfig(), brick_list=bl, origin=origin,
                                      workspace=ws)
        torch.cuda.synchronize()
    print("fill", hex(fill), "ok", st["path"], flush=True)
