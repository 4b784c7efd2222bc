"""CPU model (diagnostics): 2-D tile engine, Jacobi-PCG against the additive coarse correction on
8^2 aggregates (one damped-Jacobi coarse sweep, omega 0.8 — csrc/rwb_resident2d.cu), float64, per
64^2 tile, stop ||r|| <= tol ||S b||, with the error against the tol-1e-10 oracle.
Usage: python tools/tile_cc_model.py [random|phantom] [tol] [omega]
"""
import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import rw as orw
from paper_2509_26213_b200 import synthetic

kind = sys.argv[1] if len(sys.argv) > 1 else "random"
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
OM = float(sys.argv[3]) if len(sys.argv) > 3 else 0.8
B, AG = 64, 8
if kind == "random":
    rng = np.random.default_rng(0xC0FFEE)
    shape = (128, 192)
    vol = (rng.random(shape) * 0.3).astype(np.float32)
    seeds = np.zeros(shape, np.uint8); u = rng.random(shape)
    seeds[u < 0.05] = 1; seeds[(u >= 0.05) & (u < 0.1)] = 2
    bound = rng.random(shape).astype(np.float32).astype(np.float64)
else:
    shape = (512, 512)
    vol = synthetic.phantom(shape); seeds = synthetic.seeds(shape, "S1")
    bound = np.full(shape, 0.5)
P = orw.RWParams(tol=1e-10)
bid, nb = orw.brick_ids(shape, (B, B))
S = orw.assemble(vol, seeds, bid, nb, bound, P)
x_ref, _, _ = orw.pcg(S, bound, orw.RWParams(tol=1e-10))
EXTRA = "extra" in sys.argv
OM2 = float(sys.argv[sys.argv.index("extra") + 1]) if EXTRA and len(sys.argv) > sys.argv.index("extra") + 1 else 0.8
worst = {k: 0.0 for k in ["jacobi", "cc", "exact", "j2", "j3"]}
its = {k: 0 for k in worst}
for b in range(nb):
    by, bx = np.unravel_index(b, (shape[0] // B, shape[1] // B))
    sl = (slice(by * B, by * B + B), slice(bx * B, bx * B + B))
    unk = S.unknown[sl]
    if not unk.any(): continue
    d = np.where(unk, S.diag[sl], 1.0); s = np.where(unk, 1 / np.sqrt(d), 0)
    W = []
    for k in range(2):
        w = S.coupled[k][sl].copy(); last = [slice(None)] * 2; last[k] = slice(B - 1, B); w[tuple(last)] = 0
        a = [slice(None)] * 2; a[k] = slice(0, -1); bb = [slice(None)] * 2; bb[k] = slice(1, None)
        ws = np.zeros_like(w); ws[tuple(a)] = w[tuple(a)] * s[tuple(a)] * s[tuple(bb)]; W.append((ws, tuple(a), tuple(bb)))
    def A(x):
        y = x * unk
        for ws, a, bb in W:
            y[a] -= ws[a] * x[bb]; y[bb] -= ws[a] * x[a]
        return y
    x0 = np.where(unk, bound[sl], 0) / np.where(unk, s, 1) * unk
    rhs = S.rhs[sl] * s
    na = B // AG
    agg = lambda v: v.reshape(na, AG, na, AG).sum((1, 3))
    Pm = lambda xc: xc.repeat(AG, 0).repeat(AG, 1) * unk
    nc = na * na; Ac = np.zeros((nc, nc))
    for j in range(nc):
        e = np.zeros(nc); e[j] = 1; Ac[:, j] = agg(A(Pm(e.reshape(na, na)))).ravel()
    dg = np.diag(Ac); dci = np.where(dg > 1e-6, 1 / np.where(dg > 1e-6, dg, 1), 0)
    precs = {"jacobi": lambda r: r, "cc": lambda r: r + Pm((OM * dci * agg(r).ravel()).reshape(na, na))}
    if EXTRA:
        live = dg > 1e-6
        Acl = Ac.copy(); Acl[~live, :] = 0; Acl[:, ~live] = 0; Acl[~live, ~live] = 1
        Aci = np.linalg.inv(Acl)
        def cj(r, k):
            g = agg(r).ravel(); c = OM2 * dci * g
            for _ in range(k - 1): c = c + OM2 * dci * (g - Ac @ c)
            return Pm(c.reshape(na, na))
        precs["exact"] = lambda r: r + Pm((Aci @ agg(r).ravel()).reshape(na, na))
        precs["j2"] = lambda r: r + cj(r, 2)
        precs["j3"] = lambda r: r + cj(r, 3)
    out = [b]
    bb2 = (rhs ** 2).sum()
    for nm, pr in precs.items():
        y = x0.copy(); r = rhs - A(y); z = pr(r); p = z.copy(); rz = (r * z).sum(); it = 0
        while (r * r).sum() > tol * tol * bb2 and it < 5000:
            q = A(p); al = rz / (p * q).sum(); y += al * p; r -= al * q; z = pr(r); rzn = (r * z).sum(); p = z + rzn / rz * p; rz = rzn; it += 1
        err = np.abs(np.where(unk, y * s, 0) - np.where(unk, x_ref[sl], 0)).max()
        worst[nm] = max(worst[nm], err); its[nm] += it
        out += [nm, it, f"{err:.1e}"]
    if "v" in sys.argv[4:]: print(*out, flush=True)
print("worst", {k: f"{v:.2e}" for k, v in worst.items()}, "iterations", its)
