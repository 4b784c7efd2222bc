"""Concurrent host threads calling the library (diagnostics for the engine's worker pool)."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_26213_b200 import device, synthetic, _native
from paper_2509_26213_b200.config import RWConfig

mode = sys.argv[1] if len(sys.argv) > 1 else "solve"
nthreads, iters = 8, int(os.environ.get("MT_ITERS", "40"))
errors = []
vol_full = torch.from_numpy(synthetic.phantom((96, 96, 96))).cuda()
sd_full = torch.from_numpy(synthetic.seeds((96, 96, 96), "S1")).cuda()
par_full = torch.rand((48, 48, 48), device="cuda")


def work(tid):
    try:
        for it in range(iters):
            z0 = 32 * ((tid + it) % 2)
            lo = [max(z0 - 1, 0), 31, 31]
            hi = [z0 + 33, 65, 65]
            vol = vol_full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].contiguous()
            sd = sd_full[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].contiguous()
            if mode == "coop" or (mode == "mix" and (tid + it) % 3 == 0):
                v = vol_full[:64, :64, :64].contiguous()
                s = sd_full[:64, :64, :64].contiguous()
                prob, st = device.solve_level(v, s, (64, 64, 64), None, RWConfig())
                p = prob.cpu()
                continue
            if mode == "lod" or (mode == "mix" and (tid + it) % 3 == 1):
                l = device.lod_down(vol_full)
                p = l.cpu()
                continue
            if mode in ("window", "window_solve"):
                from paper_2509_26213_b200 import ops as rwops
                rng = np.random.default_rng(tid * 1000 + it)
                wlo = [int(rng.integers(0, 90)) for _ in range(3)]
                whi = [min(96, l + int(rng.integers(1, 40))) for l in wlo]
                plo, phi = rwops._parent_window(wlo, whi, (48, 48, 48))
                par = par_full[plo[0]:phi[0], plo[1]:phi[1], plo[2]:phi[2]].contiguous()
                win = [b - a for a, b in zip(wlo, whi)]
                fine = torch.empty(win, device="cuda")
                a64 = _native.int64_array
                _native.check(_native.lib().rwb_upsample_window_f32(
                    3, a64((48, 48, 48)), a64(plo), a64([b - a for a, b in zip(plo, phi)]), device._ptr(par),
                    a64((96, 96, 96)), a64(wlo), a64(win), device._ptr(fine), device._stream_handle()))
                if not os.environ.get("MT_NO_FULL"):
                    full = device.upsample(par_full, (96, 96, 96))
                    if not torch.equal(fine, full[wlo[0]:whi[0], wlo[1]:whi[1], wlo[2]:whi[2]]):
                        errors.append(f"window mismatch {wlo} {whi}")
                if mode == "window":
                    continue
            if mode == "ups_solve":
                bnd = device.upsample(par_full, (96, 96, 96))
            if mode == "rand_solve":
                junk = torch.rand((96, 96, 96), device="cuda")
            if mode == "upsample_only":
                bound = device.upsample(par_full, (96, 96, 96))
                continue
            bound = torch.rand(vol.shape, device="cuda")
            origin = tuple(-(a % 32) for a in lo)
            grid = device.brick_grid(vol.shape, (32, 32, 32), origin)
            idx = 0
            for hd, a, gdim in zip([z0 // 32, 1, 1], lo, grid):
                idx = idx * gdim + (hd - a // 32)
            bl = torch.tensor([idx], dtype=torch.int32, device="cuda")
            prob, st = device.solve_level(vol, sd, (32, 32, 32), bound, RWConfig(), brick_list=bl, origin=origin)
            p = prob.cpu()
    except Exception as e:  # noqa: BLE001
        errors.append(repr(e)[:300])


ts = [threading.Thread(target=work, args=(i,)) for i in range(nthreads)]
[t.start() for t in ts]
[t.join() for t in ts]
torch.cuda.synchronize()
print(mode, "errors:", len(errors), errors[:2])
