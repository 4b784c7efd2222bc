"""CPU model (diagnostics): iteration counts of the coarsest-level multigrid-PCG (rwb_mgcg.cu) and
variants, float64, on the coarsest level of a phantom hierarchy (the bench's §8(d) generator).

    python tools/mg_model.py [N] [levels] [variant ...]
      N^3 phantom, seeds S1; the coarsest level is N / 2^(levels-1) per side.
      variants: base | om=<w> | nu=<pre/post sweeps> | cs=<coarse scale> | bot=<bottom sweeps> | x0=<initial p>
                | minc=<cells of the bottom level>, combined with commas, e.g. cs=1.6,nu=2
"""
import sys
sys.path.insert(0, '/root/repo')
import numpy as np
from oracle import rw as orw, lod
from paper_2509_26213_b200 import synthetic

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
L = int(sys.argv[2]) if len(sys.argv) > 2 else 2
variants = sys.argv[3:] or ["base"]
shape = (N,) * 3
vol = synthetic.phantom(shape)
seeds = synthetic.seeds(shape, "S1")
vols = lod.lod_chain(vol, (32,) * 3, L)
sd = seeds
for _ in range(L - 1):
    sd = orw.project_seeds(sd)
v = vols[-1]
P = orw.RWParams(tol=1e-10)
bid, nb = orw.brick_ids(v.shape, v.shape)
S = orw.assemble(v, sd, bid, nb, None, P)
unk = S.unknown
s = np.where(unk, 1 / np.sqrt(np.where(unk, S.diag, 1)), 0.0)
sl = orw._sl
W = [np.zeros(v.shape) for _ in range(3)]
for k in range(3):
    a = sl(3, k, slice(0, -1)); b = sl(3, k, slice(1, None))
    W[k][a] = S.coupled[k][a] * s[a] * s[b]
print("coarsest", v.shape, "unknowns", int(unk.sum()), flush=True)


def Aop(W, dg, x):
    y = dg * x
    for k in range(3):
        a = sl(3, k, slice(0, -1)); b = sl(3, k, slice(1, None))
        y[a] -= W[k][a] * x[b]; y[b] -= W[k][a] * x[a]
    return y


def faces(W):
    f = np.zeros(W[0].shape)
    for k in range(3):
        a = sl(3, k, slice(0, -1)); b = sl(3, k, slice(1, None))
        f[a] += W[k][a]; f[b] += W[k][a]
    return f


def pad2(x):
    return np.pad(x, [(0, (-n) % 2) for n in x.shape])


def strong_mask(W, dg, TH=0.01):
    """largest strongly connected child set per 2x2x2 block (vectorised label propagation)"""
    sh = dg.shape
    dgp = pad2(dg)
    Z, Y, X = [n // 2 for n in dgp.shape]
    cells = dgp.reshape(Z, 2, Y, 2, X, 2).transpose(0, 2, 4, 1, 3, 5).reshape(Z, Y, X, 8)
    present = cells > 0
    Wp = [pad2(w) for w in W]
    Wb = [w.reshape(Z, 2, Y, 2, X, 2).transpose(0, 2, 4, 1, 3, 5).reshape(Z, Y, X, 8) for w in Wp]
    edges = []  # (i, j, strong)
    # W[k] couples along array axis k (0 = z, 1 = y, 2 = x); child index i = dz*4 + dy*2 + dx
    for i in range(8):
        for k, bit in ((0, 4), (1, 2), (2, 1)):
            if not i & bit:
                j = i | bit
                w = Wb[k][..., i]
                strong = present[..., i] & present[..., j] & (w >= TH * np.minimum(cells[..., i], cells[..., j]))
                edges.append((i, j, strong))
    lab = np.where(present, np.arange(8), 99)
    for _ in range(8):
        for i, j, st in edges:
            m = np.minimum(lab[..., i], lab[..., j])
            lab[..., i] = np.where(st, m, lab[..., i]); lab[..., j] = np.where(st, m, lab[..., j])
    counts = np.stack([(lab == c).sum(-1) for c in range(8)], -1)
    best = counts.argmax(-1)
    keep = (lab == best[..., None]) & present
    m = keep.reshape(Z, Y, X, 2, 2, 2).transpose(0, 3, 1, 4, 2, 5).reshape(dgp.shape)
    return m[:sh[0], :sh[1], :sh[2]]


def agg(x, sh):
    x = np.pad(x, [(0, 2 * c - n) for c, n in zip(sh, x.shape)])
    return x.reshape(sh[0], 2, sh[1], 2, sh[2], 2).sum((1, 3, 5))


def coarsen(W, leak, dg):
    m = strong_mask(W, dg); sh = tuple((n + 1) // 2 for n in leak.shape)
    lk = leak.copy()
    for k in range(3):
        a = sl(3, k, slice(0, -1)); b = sl(3, k, slice(1, None))
        lk[a] += W[k][a] * (~m[b]); lk[b] += W[k][a] * (~m[a])
    lk = lk * m; Wc = []
    for k in range(3):
        mm = np.zeros(W[k].shape); s_ = [slice(None)] * 3; s_[k] = slice(1, None, 2); s_ = tuple(s_)
        a = sl(3, k, slice(0, -1)); b = sl(3, k, slice(1, None))
        both = np.zeros(W[k].shape, bool); both[a] = m[a] & m[b]
        mm[s_] = (W[k] * both)[s_]; Wc.append(agg(mm, sh))
    lkc = agg(lk, sh); return Wc, lkc, lkc + faces(Wc), m


def P_(x, sh):
    y = x.repeat(2, 0).repeat(2, 1).repeat(2, 2); return y[:sh[0], :sh[1], :sh[2]]


def build(minc):
    dg0 = unk.astype(float); leak0 = np.where(unk, 1.0 - faces(W), 0.0)
    levels = [(W, leak0, dg0, None)]
    while np.prod(levels[-1][1].shape) > minc:
        Wc, lk, dg, m = coarsen(*levels[-1][:3]); levels[-1] = levels[-1][:3] + (m,); levels.append((Wc, lk, dg, None))
    return levels


def run(opts):
    om, nu, cs, bot, minc = opts.get("om", 0.8), int(opts.get("nu", 1)), opts.get("cs", 1.0), int(opts.get("bot", 8)), int(opts.get("minc", 64))
    levels = build(minc)
    tg = int(opts.get("tg", 0))  # > 0: exact solve on level tg (two-grid model when 1)
    if tg:
        import scipy.sparse as sp
        import scipy.sparse.linalg as spl
        W_, lk, dg, _ = levels[tg]
        sh = dg.shape; n = dg.size; idx = np.arange(n).reshape(sh)
        rows, cols, vals = [np.arange(n)], [np.arange(n)], [np.where(dg > 0, dg, 1.0).ravel()]
        for k in range(3):
            a = sl(3, k, slice(0, -1)); b = sl(3, k, slice(1, None))
            rows += [idx[a].ravel(), idx[b].ravel()]; cols += [idx[b].ravel(), idx[a].ravel()]
            vals += [-W_[k][a].ravel(), -W_[k][a].ravel()]
        A = sp.csc_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))
        lu = spl.splu(A)

    def vcycle(c, b):
        W_, lk, dg, m = levels[c]; dinv = np.where(dg > 0, 1 / np.where(dg > 0, dg, 1), 0)
        if tg and c == tg:
            return lu.solve(b.ravel()).reshape(b.shape) * (dg > 0)
        if c == len(levels) - 1:
            x = om * dinv * b
            for _ in range(bot - 1): x = x + om * dinv * (b - Aop(W_, dg, x))
            return x
        x = om * dinv * b
        for _ in range(nu - 1): x = x + om * dinv * (b - Aop(W_, dg, x))
        res = b - Aop(W_, dg, x)
        xc = vcycle(c + 1, agg(res * m, levels[c + 1][1].shape))
        x = x + cs * P_(xc, b.shape) * m
        for _ in range(nu): x = x + om * dinv * (b - Aop(W_, dg, x))
        return x

    b = np.where(unk, S.rhs * s, 0); bb = float((b ** 2).sum())
    dg0 = unk.astype(float)
    x0 = float(opts.get("x0", 0.0))  # initial probability of the unknowns
    y = np.where(unk, x0 / np.where(unk, s, 1.0), 0.0)
    r = b - Aop(W, dg0, y); z = vcycle(0, r); p = z.copy(); rz = float((r * z).sum()); it = 0
    while float((r ** 2).sum()) > 1e-12 * bb and it < 500:
        q = Aop(W, dg0, p); al = rz / float((p * q).sum()); y += al * p; r -= al * q
        z = vcycle(0, r); rzn = float((r * z).sum()); p = z + rzn / rz * p; rz = rzn; it += 1
    return it, len(levels)


for var in variants:
    opts = {}
    if var != "base":
        for kv in var.split(","):
            k, val = kv.split("="); opts[k] = float(val)
    it, nl = run(opts)
    print(var, "levels", nl, "iterations", it, flush=True)
