"""CPU baseline of a large hierarchy by the BASELINE.md §4 plan (test / benchmark infrastructure).

For config 4 (1024^3, 4 levels) a full float64 oracle run takes hours, so the CPU throughput is
measured the way BASELINE.md §4 specifies: "coarsest level timed fully; a fixed random sample of
bricks per finer level timed, then extrapolated by brick count (labelled 'extrapolated')".  All
work runs on the host's cores with the float64 numpy oracle (`oracle/rw.py`, `oracle/lod.py`):

* setup: the full LOD pyramid and seed levels of the real input (slab-parallel), so the coarsest
  level is the real one; the coarsest level's whole Jacobi-PCG solve (tol as the GPU's),
  slab-parallel over the cores (`solve_whole_threaded`), timed in full (`top_full_seconds`); and
  `chains` fixed random sample positions;
* per step (timed, every part measured in that step):
  - the LOD pyramid and the seed projections on a level-0 slab of `slab_planes` planes (with the
    matching slabs of the coarser levels), scaled by the level-0 plane count;
  - the coarsest solve's first `top_sample_iterations` iterations (assembly included), scaled to
    the setup's full iteration count;
  - the prolongation of the coarsest solution to the next level, scaled by voxels to every level;
  - `chains` brick chains on `chains` threads: each chain solves a 2x2x2 block of bricks of the
    level below the coarsest (bound = upsampled coarsest solution), then the 2x2x2 block of its
    interior children one level finer (bound = upsampled block solution: the children's
    prolongation taps lie inside the solved block), and so on down to level 0 — 8 real bricks per
    level per chain, each with its true Dirichlet halo;  level k costs
    (measured wall time of the chain wave) x n_bricks_k / (8 x chains), i.e. the throughput of
    `chains` cores kept busy, the same as a full level run on that many cores.
  The extrapolated time is the sum; voxels/s = level-0 voxels / that time.
"""

from __future__ import annotations

import math
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import lod as olod
from . import rw as orw


# ---------------------------------------------------------------------------
# slab-parallel primitives (identical per-element arithmetic to the serial oracle)


def _slabs(n, parts):
    parts = max(1, min(parts, n))
    return [(n * i // parts, n * (i + 1) // parts) for i in range(parts)]


def lod_down_threaded(level: np.ndarray, pool, parts: int, slab: int = 16) -> np.ndarray:
    """`lod.lod_down`, coarse planes split over threads (bit-identical, `lod_down_slabbed`)."""
    level = np.asarray(level, dtype=np.float32)
    n = level.shape[0]
    m = -(-n // 2)
    out = np.empty((m,) + tuple(-(-s // 2) for s in level.shape[1:]), dtype=np.float32)

    def run(rng):
        j0, j1 = rng
        for a in range(j0, j1, slab):
            b = min(a + slab, j1)
            f0, f1 = max(2 * a - 1, 0), min(2 * b + 1, n)
            conv = olod.separable_conv_clamp(level[f0:f1], [olod.SMOOTHING_KERNEL] * level.ndim).astype(np.float32)
            keep = conv[2 * a - f0:min(2 * b, n) - f0]
            out[a:b] = olod.pairwise_mean(keep).astype(np.float32)

    list(pool.map(run, _slabs(m, parts)))
    return out


def project_seeds_threaded(seeds: np.ndarray, pool, parts: int) -> np.ndarray:
    n = seeds.shape[0]
    m = -(-n // 2)
    out = np.empty((m,) + tuple(-(-s // 2) for s in seeds.shape[1:]), dtype=np.uint8)

    def run(rng):
        j0, j1 = rng
        out[j0:j1] = orw.project_seeds(seeds[2 * j0:min(2 * j1, n)])

    list(pool.map(run, _slabs(m, parts)))
    return out


def solve_whole_threaded(volume, seeds, params: orw.RWParams, pool, parts: int, iterations: int | None = None):
    """Whole-level (single brick) Jacobi-PCG of `rw.pcg` with the stencil, the dot products and
    the vector updates split into z-slabs over the pool (float64; the slab partial sums are added
    in slab order).  `iterations`: stop after that many (a timing sample).  Returns (prob,
    iterations)."""
    shape = np.shape(volume)
    bid, nb = orw.brick_ids(shape, shape)
    sys_ = orw.assemble(volume, seeds, bid, nb, None, params)
    nd = len(shape)
    nz = shape[0]
    unk = sys_.unknown
    diag = sys_.diag
    cpl = sys_.coupled
    dinv = np.where(unk, 1.0 / diag, 0.0)
    b = sys_.rhs
    sl = _slabs(nz, parts)
    x = np.zeros(shape)
    r = b.copy()
    z = np.empty(shape)
    p = np.empty(shape)
    q = np.empty(shape)

    def lap(a, e, src, dst):
        xs = src[a:e]
        y = diag[a:e] * xs
        hi = min(e, nz - 1)
        if hi > a:
            y[:hi - a] -= cpl[0][a:hi] * src[a + 1:hi + 1]
        lo = max(a, 1)
        if e > lo:
            y[lo - a:] -= cpl[0][lo - 1:e - 1] * src[lo - 1:e - 1]
        for k in range(1, nd):
            s0 = orw._sl(nd, k, slice(0, -1))
            s1 = orw._sl(nd, k, slice(1, None))
            ck = cpl[k][a:e]
            y[s0] -= ck[s0] * xs[s1]
            y[s1] -= ck[s0] * xs[s0]
        dst[a:e] = np.where(unk[a:e], y, 0.0)

    def par(fn):
        return list(pool.map(fn, sl))

    bb = sum(par(lambda s: float(np.dot(b[s[0]:s[1]].ravel(), b[s[0]:s[1]].ravel()))))
    if bb <= 0.0:
        return np.where(unk, 0.0, sys_.dvals), 0
    tol2 = params.tol * params.tol

    def init(s):
        a, e = s
        z[a:e] = dinv[a:e] * r[a:e]
        p[a:e] = z[a:e]
        return float(np.dot(r[a:e].ravel(), z[a:e].ravel())), float(np.dot(r[a:e].ravel(), r[a:e].ravel()))

    parts_ = par(init)
    rz = sum(v[0] for v in parts_)
    rr = sum(v[1] for v in parts_)
    it = 0
    cap = params.max_iter if iterations is None else min(params.max_iter, iterations)
    while rr > tol2 * bb and it < cap:
        def spmv(s):
            lap(s[0], s[1], p, q)
            return float(np.dot(p[s[0]:s[1]].ravel(), q[s[0]:s[1]].ravel()))

        pq = sum(par(spmv))
        alpha = rz / pq if pq != 0 else 0.0

        def upd(s):
            a, e = s
            x[a:e] += alpha * p[a:e]
            r[a:e] -= alpha * q[a:e]
            z[a:e] = dinv[a:e] * r[a:e]
            return float(np.dot(r[a:e].ravel(), z[a:e].ravel())), float(np.dot(r[a:e].ravel(), r[a:e].ravel()))

        parts_ = par(upd)
        rz_new = sum(v[0] for v in parts_)
        rr = sum(v[1] for v in parts_)
        beta = rz_new / rz if rz != 0 else 0.0
        rz = rz_new

        def dirn(s):
            a, e = s
            p[a:e] = z[a:e] + beta * p[a:e]

        par(dirn)
        it += 1
    return np.where(unk, x, sys_.dvals), it


# ---------------------------------------------------------------------------
# brick chains


def _block_solve(vol, seeds, parent_full, parent_z0, level_shape, brick, lo, hi, params):
    """Solve the bricks of the fine block [lo, hi) (global coords, whole bricks) of a level of
    shape `level_shape`, bound = prolongation of `parent_full` (a parent window whose first
    global corner is `parent_z0`, NaN where unknown).  Returns the block's probabilities."""
    nd = len(level_shape)
    rlo = [max(a - 1, 0) for a in lo]
    rhi = [min(b + 1, n) for b, n in zip(hi, level_shape)]
    sel = tuple(slice(a, b) for a, b in zip(rlo, rhi))
    # prolongation taps in global coordinates, evaluated on the parent window (shift by its corner)
    bound = np.empty([b - a for a, b in zip(rlo, rhi)])
    out = None
    src = parent_full
    for dim in range(nd):
        n = level_shape[dim]
        m = -(-n // 2)
        g = np.arange(rlo[dim], rhi[dim], dtype=np.float64)
        c = g / 2.0 - 0.25
        fl = np.floor(c)
        t = c - fl
        i0 = np.clip(fl.astype(np.int64), 0, m - 1) - parent_z0[dim]
        i1 = np.clip(fl.astype(np.int64) + 1, 0, m - 1) - parent_z0[dim]
        if min(i0.min(), i1.min()) < 0 or max(i0.max(), i1.max()) >= src.shape[dim]:
            raise RuntimeError("brick chain read a parent value outside its solved block")
        shp = [1] * nd
        shp[dim] = len(g)
        t = t.reshape(shp)
        src = np.take(src, i0, axis=dim) * (1.0 - t) + np.take(src, i1, axis=dim) * t
        out = src
    bound[...] = out
    mask = np.zeros(bound.shape, bool)
    mask[tuple(slice(a - r, b - r) for a, b, r in zip(lo, hi, rlo))] = True
    res = orw.solve_level(vol[sel], seeds[sel], brick, bound, params, solve_mask=mask, origin=tuple(rlo))
    return res.prob[tuple(slice(a - r, b - r) for a, b, r in zip(lo, hi, rlo))]


def run_chain(vols, seeds, top_prob, brick, params, start):
    """One chain: start = brick coordinates (level L-2) of the 2x2x2 block's first brick."""
    L = len(vols)
    parent, pz0 = top_prob, (0,) * vols[0].ndim
    pos = list(start)
    times = []
    for k in range(L - 2, -1, -1):
        shape = vols[k].shape
        lo = [p * b for p, b in zip(pos, brick)]
        hi = [min(a + 2 * b, n) for a, b, n in zip(lo, brick, shape)]
        t0 = time.perf_counter()
        blk = _block_solve(vols[k], seeds[k], parent, pz0, shape, brick, lo, hi, params)
        times.append(time.perf_counter() - t0)
        parent, pz0 = blk, tuple(lo)
        pos = [2 * p + 1 for p in pos]  # the interior children one level finer
    return times


def chain_starts(shapes, brick, chains, seed=0xC0FFEE):
    """Fixed random block positions at level L-2 whose descendant blocks stay interior."""
    rng = np.random.default_rng(seed)
    L = len(shapes)
    grid = [-(-n // b) for n, b in zip(shapes[L - 2], brick)]
    out = []
    for _ in range(chains):
        out.append(tuple(int(rng.integers(0, max(g - 1, 1))) for g in grid))
    return out


class C4Baseline:
    """Setup once (full pyramid, the coarsest solve timed in full, sample positions); `step()`
    times one extrapolated run."""

    def __init__(self, volume, seeds, brick, levels, params: orw.RWParams, cores=None, chains=None,
                 slab_planes=128, top_sample_iterations=40):
        self.cores = cores or len(os.sched_getaffinity(0))
        self.chains = chains or self.cores
        self.pool = ThreadPoolExecutor(max_workers=self.cores)
        self.brick, self.params = tuple(brick), params
        self.vols = [np.asarray(volume, dtype=np.float32)]
        self.seeds = [np.asarray(seeds, dtype=np.uint8)]
        for _ in range(levels - 1):
            self.vols.append(lod_down_threaded(self.vols[-1], self.pool, self.cores))
            self.seeds.append(project_seeds_threaded(self.seeds[-1], self.pool, self.cores))
        self.shapes = [v.shape for v in self.vols]
        self.starts = chain_starts(self.shapes, self.brick, self.chains)
        self.slab_planes = min(slab_planes, self.shapes[0][0])
        # the coarsest level solved (and timed) in full once: its solution bounds the chains, its
        # iteration count scales the per-step timing sample
        t0 = time.perf_counter()
        self.top, self.top_iterations = solve_whole_threaded(self.vols[-1], self.seeds[-1], params, self.pool,
                                                             self.cores)
        self.top_full_seconds = time.perf_counter() - t0
        self.top_sample = max(1, min(top_sample_iterations, self.top_iterations))

    def step(self):
        L = len(self.vols)
        parts = {}
        # LOD + seed projection on a level-0 slab (and the matching coarser slabs), scaled
        t0 = time.perf_counter()
        v, s = self.vols[0][:self.slab_planes], self.seeds[0][:self.slab_planes]
        for _ in range(L - 1):
            v = lod_down_threaded(v, self.pool, self.cores)
            s = project_seeds_threaded(s, self.pool, self.cores)
        parts["lod_and_seeds"] = (time.perf_counter() - t0) * self.shapes[0][0] / self.slab_planes
        # coarsest level: a sample of its iterations (assembly included), scaled to the full count
        if self.top_iterations > 0:
            t0 = time.perf_counter()
            solve_whole_threaded(self.vols[-1], self.seeds[-1], self.params, self.pool, self.cores,
                                 iterations=self.top_sample)
            parts["coarsest"] = (time.perf_counter() - t0) * self.top_iterations / self.top_sample
        else:
            parts["coarsest"] = self.top_full_seconds
        # prolongation, measured on the coarsest -> next level, scaled by voxels
        t0 = time.perf_counter()
        orw.upsample_linear(self.top, self.shapes[-2])
        dt = time.perf_counter() - t0
        parts["prolongation"] = dt * sum(math.prod(self.shapes[k]) for k in range(L - 1)) / math.prod(self.shapes[-2])
        # brick chains, one per thread
        t0 = time.perf_counter()
        per = list(self.pool.map(lambda st: run_chain(self.vols, self.seeds, self.top, self.brick, self.params, st),
                                 self.starts))
        wave = time.perf_counter() - t0
        # level k's share of the wave by its summed per-chain times
        lvl_t = [sum(p[i] for p in per) for i in range(L - 1)]  # i = 0 -> level L-2
        tot = sum(lvl_t) or 1.0
        for i in range(L - 1):
            k = L - 2 - i
            nb = math.prod(-(-n // b) for n, b in zip(self.shapes[k], self.brick))
            sampled = (2 ** len(self.shapes[k])) * self.chains
            parts[f"level{k}_bricks"] = wave * (lvl_t[i] / tot) * nb / sampled
        total = sum(parts.values())
        return total, parts

    def close(self):
        self.pool.shutdown()
