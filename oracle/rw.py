"""Float64 CPU restatement of the hierarchical random walker (test infrastructure only).

**Parity unpinned against the reference**: the reference repository contains
no random-walker code (`SPEC.md:8, 425, 802`; Palace's own implementation is
not vendored, only cited at `PAPER.md:36`).  The maths follows Grady 2006
(`PAPER.md:159`, "random walker algorithm for image segmentation") and the
brick-wise coarse-to-fine scheme of Drees et al. 2022 (`PAPER.md:417-423`).
Every discretionary rule is pinned here and mirrored by the CUDA path
(DESIGN.md §3 lists them):

* weights: forward edge (i, i+e_k) of the 2d/3d grid graph gets
  ``max(exp(-beta * (I_i - I_j)^2), min_weight)``; no edges leave the volume
  (Neumann border).  Intensities are the float32 LOD levels
  (`oracle.lod`, = `ops.build_lod`, `ops.py:714-727`).
* seeds: U8 labels, 0 = unseeded, 1 = foreground (value 1), 2 = background
  (value 0).  A coarse voxel inherits label 1 (2) when any of its <= 2^d
  children (the `downsample_mean` block, `ops.py:629-636`) is 1 (2) and none
  is 2 (1); conflicting or unseeded blocks stay 0.
* coarsest level: one whole-level Dirichlet problem, x0 = 0.
* finer levels: bricks = the level's chunk grid (`model.py:125-170`).  Each
  brick is an independent Dirichlet problem: its unseeded voxels are the
  unknowns; seeds inside it and every voxel outside it are Dirichlet nodes
  whose value is the seed value, else the upsampled parent solution U.
  x0 = U.
* upsampling: cell-centred multilinear, fine index g samples parent
  coordinate g/2 - 1/4 (taps 1/4, 3/4), clamped at the border — the
  footprint-centre convention of `procedural_lod` (`ops.py:758`).
* solver: Jacobi-preconditioned CG, stop when ||r||_2 <= tol * ||b||_2 per
  brick (b = Dirichlet right-hand side); a brick with ||b|| = 0 has the exact
  solution 0.
* labels: ``p > 0.5`` as U8 (`cast_array` semantics, `ops.py:44-52`).

The level-wide formulation solves all bricks of a level at once as one
block-diagonal system (couplings across brick faces removed), with
per-brick CG scalars; `tests/test_oracle_rw.py` checks it brick by brick
against `scipy.sparse.linalg.spsolve` on an explicitly assembled Laplacian.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import lod

SEED_NONE, SEED_FG, SEED_BG = 0, 1, 2


@dataclass(frozen=True)
class RWParams:
    beta: float = 100.0
    min_weight: float = 1e-6
    tol: float = 1e-10
    max_iter: int = 10_000


@dataclass
class LevelResult:
    prob: np.ndarray
    iterations: np.ndarray  # per brick
    converged: np.ndarray  # per brick, bool
    info: dict = field(default_factory=dict)


# ---------------------------------------------------------------------------
# elementary operators


def _sl(ndim, dim, s):
    out = [slice(None)] * ndim
    out[dim] = s
    return tuple(out)


def edge_weights(volume: np.ndarray, beta: float, min_weight: float) -> list:
    """Forward-edge weights, one array per dimension, shaped like the volume.

    ``w[k][i]`` is the weight of edge (i, i + e_k); entries whose neighbour
    lies outside the volume are 0 (no edge).
    """
    vol = np.asarray(volume, dtype=np.float64)
    out = []
    for k in range(vol.ndim):
        w = np.zeros(vol.shape, dtype=np.float64)
        if vol.shape[k] > 1:
            a = _sl(vol.ndim, k, slice(0, -1))
            b = _sl(vol.ndim, k, slice(1, None))
            d = vol[a] - vol[b]
            w[a] = np.maximum(np.exp(-beta * d * d), min_weight)
        out.append(w)
    return out


def _block_reduce_any(mask: np.ndarray) -> np.ndarray:
    out = mask
    for dim in range(out.ndim):
        n = out.shape[dim]
        even = n - n % 2
        paired = out[_sl(out.ndim, dim, slice(0, even, 2))] | out[_sl(out.ndim, dim, slice(1, even, 2))]
        if n % 2:
            paired = np.concatenate([paired, out[_sl(out.ndim, dim, slice(n - 1, n))]], axis=dim)
        out = paired
    return out


def project_seeds(seeds: np.ndarray) -> np.ndarray:
    """Seed labels of the next coarser level (conflicts -> unseeded)."""
    fg = _block_reduce_any(seeds == SEED_FG)
    bg = _block_reduce_any(seeds == SEED_BG)
    out = np.zeros(fg.shape, dtype=np.uint8)
    out[fg & ~bg] = SEED_FG
    out[bg & ~fg] = SEED_BG
    return out


def upsample_linear(parent: np.ndarray, fine_shape) -> np.ndarray:
    """Cell-centred multilinear prolongation, clamped (float64)."""
    out = np.asarray(parent, dtype=np.float64)
    for dim, n in enumerate(fine_shape):
        m = out.shape[dim]
        if -(-n // 2) != m:
            raise ValueError(f"fine size {n} is not a 2x refinement of {m}")
        g = np.arange(n, dtype=np.float64)
        c = g / 2.0 - 0.25
        lo = np.floor(c)
        t = c - lo
        i0 = np.clip(lo.astype(np.int64), 0, m - 1)
        i1 = np.clip(lo.astype(np.int64) + 1, 0, m - 1)
        shape = [1] * out.ndim
        shape[dim] = n
        t = t.reshape(shape)
        out = np.take(out, i0, axis=dim) * (1.0 - t) + np.take(out, i1, axis=dim) * t
    return out


def upsample_linear_window(parent: np.ndarray, fine_shape, lo, hi) -> np.ndarray:
    """Fine voxels [lo, hi) of `upsample_linear(parent, fine_shape)` — the same float64
    operations per element (the same taps in the same dimension order), so identical to slicing
    the full prolongation; only the parent planes the window reads are touched."""
    out = None
    src = parent
    for dim, n in enumerate(fine_shape):
        m = parent.shape[dim]
        if -(-n // 2) != m:
            raise ValueError(f"fine size {n} is not a 2x refinement of {m}")
        g = np.arange(lo[dim], hi[dim], dtype=np.float64)
        c = g / 2.0 - 0.25
        fl = np.floor(c)
        t = c - fl
        i0 = np.clip(fl.astype(np.int64), 0, m - 1)
        i1 = np.clip(fl.astype(np.int64) + 1, 0, m - 1)
        if dim == 0:  # cut the parent to the planes this window reads before anything is float64
            a, b = int(min(i0.min(), i1.min())), int(max(i0.max(), i1.max())) + 1
            src = np.asarray(parent[a:b], dtype=np.float64)
            i0, i1 = i0 - a, i1 - a
        shape = [1] * parent.ndim
        shape[dim] = len(g)
        t = t.reshape(shape)
        src = np.take(src, i0, axis=dim) * (1.0 - t) + np.take(src, i1, axis=dim) * t
        out = src
    return out


def solve_brick(volume, seeds, parent_prob, brick, h, params: RWParams) -> tuple:
    """The oracle's solution of ONE brick `h` (grid position) of a finer level, given the
    parent level's probabilities (`parent_prob`, e.g. the ones the GPU computed): its box plus
    a one-voxel Dirichlet halo is cut out of the level, bounded by the windowed prolongation of
    the parent, and solved exactly as `solve_level` solves it inside the whole level (the brick
    is an independent Dirichlet problem).  Returns (box slices, probabilities over the box)."""
    nd = volume.ndim
    b0 = [int(h[d]) * brick[d] for d in range(nd)]
    b1 = [min(b0[d] + brick[d], volume.shape[d]) for d in range(nd)]
    lo = [max(b0[d] - 1, 0) for d in range(nd)]
    hi = [min(b1[d] + 1, volume.shape[d]) for d in range(nd)]
    sl = tuple(slice(l, e) for l, e in zip(lo, hi))
    bound = upsample_linear_window(parent_prob, volume.shape, lo, hi)
    inside = np.zeros(bound.shape, dtype=bool)
    inside[tuple(slice(a - l, b - l) for a, b, l in zip(b0, b1, lo))] = True
    res = solve_level(np.asarray(volume[sl]), np.asarray(seeds[sl]), brick, bound, params, solve_mask=inside,
                      origin=tuple(lo))
    box = tuple(slice(a, b) for a, b in zip(b0, b1))
    return box, res.prob[tuple(slice(a - l, b - l) for a, b, l in zip(b0, b1, lo))], res


def seed_values(seeds: np.ndarray) -> np.ndarray:
    return (seeds == SEED_FG).astype(np.float64)


def labels_from_prob(prob: np.ndarray) -> np.ndarray:
    return (np.asarray(prob) > 0.5).astype(np.uint8)


# ---------------------------------------------------------------------------
# block-diagonal Dirichlet system of one level


def brick_ids(shape, brick, origin=None) -> tuple:
    """Row-major brick index of every voxel and the brick count (model.py:138-146).

    `origin` shifts the global coordinates of a sub-array so slabs cut out of
    a level keep the level's brick grid; ids are renumbered from 0.
    """
    origin = origin or (0,) * len(shape)
    coords = [(np.arange(s) + o) // b for s, b, o in zip(shape, brick, origin)]
    grid = [int(c[-1] - c[0]) + 1 for c in coords]
    bid = np.zeros(shape, dtype=np.int64)
    for dim, c in enumerate(coords):
        c = (c - c[0]).reshape([-1 if i == dim else 1 for i in range(len(shape))])
        bid = bid * grid[dim] + c
    return bid, int(np.prod(grid))


@dataclass
class System:
    unknown: np.ndarray  # bool
    diag: np.ndarray  # float64, all incident edge weights (unknown rows)
    coupled: list  # per dim: forward weight where both ends are unknowns of one brick
    rhs: np.ndarray  # Dirichlet right-hand side (unknown rows)
    dvals: np.ndarray  # Dirichlet values (seeds, or bound) for every voxel
    bid: np.ndarray
    nbricks: int


def assemble(volume, seeds, bid, nbricks, bound, params: RWParams, solve_mask=None) -> System:
    """Block-diagonal Dirichlet system L_UU x = rhs over all bricks of a level."""
    vol = np.asarray(volume, dtype=np.float32)
    seeds = np.asarray(seeds, dtype=np.uint8)
    nd = vol.ndim
    if bound is None and nbricks > 1:
        raise ValueError("brick-wise solve needs boundary values from the parent level")
    w = edge_weights(vol, params.beta, params.min_weight)
    unknown = seeds == SEED_NONE
    if solve_mask is not None:
        unknown = unknown & solve_mask
    dvals = seed_values(seeds)
    if bound is not None:
        dvals = np.where(seeds == SEED_NONE, np.asarray(bound, dtype=np.float64), dvals)
    diag = np.zeros(vol.shape, dtype=np.float64)
    rhs = np.zeros(vol.shape, dtype=np.float64)
    coupled = []
    for k in range(nd):
        a = _sl(nd, k, slice(0, -1))
        b = _sl(nd, k, slice(1, None))
        wk = w[k][a]
        diag[a] += wk
        diag[b] += wk
        same = bid[a] == bid[b]
        ua, ub = unknown[a], unknown[b]
        c = np.zeros(vol.shape, dtype=np.float64)
        c[a] = wk * (ua & ub & same)
        coupled.append(c)
        # Dirichlet neighbours: seeded, outside the solve mask, or in another brick
        rhs[a] += wk * dvals[b] * (ua & ~(ub & same))
        rhs[b] += wk * dvals[a] * (ub & ~(ua & same))
    diag = np.where(unknown, diag, 1.0)
    rhs = np.where(unknown, rhs, 0.0)
    return System(unknown, diag, coupled, rhs, dvals, bid, nbricks)


def apply_laplacian(sys_: System, x: np.ndarray) -> np.ndarray:
    """L_UU x on unknown rows (x must be zero on Dirichlet nodes)."""
    nd = x.ndim
    y = sys_.diag * x
    for k, c in enumerate(sys_.coupled):
        a = _sl(nd, k, slice(0, -1))
        b = _sl(nd, k, slice(1, None))
        y[a] -= c[a] * x[b]
        y[b] -= c[a] * x[a]
    return np.where(sys_.unknown, y, 0.0)


def pcg(sys_: System, x0, params: RWParams):
    """Jacobi-PCG over all bricks at once with per-brick scalars (float64)."""
    unk = sys_.unknown
    bid = sys_.bid.ravel()
    nb = sys_.nbricks

    def bsum(v):
        return np.bincount(bid, weights=v.ravel(), minlength=nb)

    x = np.where(unk, np.asarray(x0, dtype=np.float64), 0.0) if x0 is not None else np.zeros(unk.shape)
    b = sys_.rhs
    bb = bsum(b * b)
    zero_bricks = bb <= 0.0
    x[zero_bricks[sys_.bid] & unk] = 0.0
    r = np.where(unk, b - apply_laplacian(sys_, x), 0.0)
    dinv = np.where(unk, 1.0 / sys_.diag, 0.0)
    tol2 = params.tol * params.tol
    rr = bsum(r * r)
    active = (~zero_bricks) & (rr > tol2 * bb)
    iters = np.zeros(nb, dtype=np.int64)
    z = dinv * r
    p = z.copy()
    rz = bsum(r * z)
    with np.errstate(divide="ignore", invalid="ignore"):
        for _ in range(params.max_iter):
            if not active.any():
                break
            q = apply_laplacian(sys_, p)
            pq = bsum(p * q)
            alpha = np.where(active, rz / np.where(pq == 0, 1.0, pq), 0.0)
            x += alpha[sys_.bid] * p
            r -= alpha[sys_.bid] * q
            rr = bsum(r * r)
            iters += active
            active &= rr > tol2 * bb
            z = dinv * r
            rz_new = bsum(r * z)
            beta = np.where(active, rz_new / np.where(rz == 0, 1.0, rz), 0.0)
            rz = rz_new
            p = z + beta[sys_.bid] * p
    converged = ~active
    return x, iters, converged


def solve_level(volume, seeds, brick, bound, params: RWParams, solve_mask=None,
                origin=None) -> LevelResult:
    """One level: whole-level solve when `brick` covers it, else brick-wise."""
    bid, nb = brick_ids(np.shape(volume), brick, origin)
    sys_ = assemble(volume, seeds, bid, nb, bound, params, solve_mask)
    x, iters, conv = pcg(sys_, bound, params)
    prob = np.where(sys_.unknown, x, sys_.dvals)
    return LevelResult(prob, iters, conv)


def solve_level_threaded(volume, seeds, brick, bound, params: RWParams, workers=None) -> LevelResult:
    """Same result as `solve_level`, split into tiles of bricks along dims 0 (and 1 when there
    are more workers than brick slabs along dim 0).

    Bricks are independent given `bound`, so each tile (plus a one-voxel Dirichlet halo on each
    cut side) is solved on its own thread; numpy releases the GIL inside its array kernels, the
    way the reference engine runs chunk kernels on its worker pool (`engine.py:398-400, 866-875`).
    """
    workers = workers or len(os.sched_getaffinity(0))
    shape = volume.shape
    nd = volume.ndim
    nslab = [-(-shape[d] // brick[d]) for d in range(min(nd, 2))]
    if bound is None or workers == 1 or (nslab[0] == 1 and (nd < 2 or nslab[1] == 1)):
        return solve_level(volume, seeds, brick, bound, params)
    parts = [min(workers, nslab[0])]
    if nd >= 2:
        parts.append(min(nslab[1], max(1, workers // parts[0])))
    spans = []
    for d, k in enumerate(parts):
        per = -(-nslab[d] // k)
        spans.append([(s * brick[d], min((s + per) * brick[d], shape[d])) for s in range(0, nslab[d], per)])
    tiles = [(a,) for a in spans[0]] if len(spans) == 1 else [(a, b) for a in spans[0] for b in spans[1]]

    def run(tile):
        lo = [max(0, a - 1) for a, _ in tile]
        hi = [min(shape[d], b + 1) for d, (_, b) in enumerate(tile)]
        sl = tuple(slice(l, h) for l, h in zip(lo, hi))
        inside = np.ones(tuple(h - l for l, h in zip(lo, hi)) + shape[len(tile):], dtype=bool)
        for d, (a, b) in enumerate(tile):
            keep = np.zeros(hi[d] - lo[d], dtype=bool)
            keep[a - lo[d]:b - lo[d]] = True
            inside &= keep.reshape([-1 if i == d else 1 for i in range(nd)])
        origin = tuple(lo) + (0,) * (nd - len(tile))
        res = solve_level(volume[sl], seeds[sl], brick, bound[sl], params, solve_mask=inside, origin=origin)
        return tile, lo, res

    prob = np.empty(shape, dtype=np.float64)
    with ThreadPoolExecutor(max_workers=len(tiles)) as pool:
        results = list(pool.map(run, tiles))
    its = []
    for tile, lo, res in results:
        dst = tuple(slice(a, b) for a, b in tile)
        src = tuple(slice(a - l, b - l) for (a, b), l in zip(tile, lo))
        prob[dst] = res.prob[src]
        its.append(res.iterations)
    return LevelResult(prob, np.concatenate(its), np.zeros(0, bool), {"tiles": len(tiles)})


# ---------------------------------------------------------------------------
# hierarchical driver


@dataclass
class HierarchyResult:
    prob: list  # per level, float64, level 0 finest
    seeds: list
    volumes: list
    iterations: list  # per level, per brick
    labels: np.ndarray


def decided_bricks(bound, seeds, brick, eps: float) -> np.ndarray:
    """The optional brick-skip rule of the hierarchical scheme (Drees et al. 2022, `PAPER.md:419`,
    SURVEY.md §8(a) N5): a brick is skipped — its values are the upsampled parent, seeds exact —
    when every value its solve would read, the upsampled parent over the brick and its one-voxel
    halo, is within `eps` of 0 or 1 (seeded voxels count as decided).  Per brick, row-major."""
    amb = np.minimum(bound, 1.0 - bound)
    amb = np.where(np.asarray(seeds) != SEED_NONE, 0.0, amb)
    grid = [-(-n // b) for n, b in zip(amb.shape, brick)]
    out = np.zeros(grid, dtype=bool)
    for h in np.ndindex(*grid):
        sl = tuple(slice(max(i * b - 1, 0), min((i + 1) * b + 1, n)) for i, b, n in zip(h, brick, amb.shape))
        out[h] = amb[sl].max() < eps
    return out.reshape(-1)


def hierarchical_random_walker(volume, seeds, brick, levels=None, params: RWParams = RWParams(),
                               threads: int | None = 1, skip_eps: float | None = None) -> HierarchyResult:
    """Coarsest level whole, then every finer level brick by brick (with `skip_eps`, bricks whose
    parent is decided keep the upsampled parent: `decided_bricks`)."""
    vols = lod.lod_chain(volume, brick, levels)
    seed_levels = [np.asarray(seeds, dtype=np.uint8)]
    for _ in range(len(vols) - 1):
        seed_levels.append(project_seeds(seed_levels[-1]))
    nlev = len(vols)
    probs = [None] * nlev
    iters = [None] * nlev
    top = solve_level(vols[-1], seed_levels[-1], vols[-1].shape, None, params)
    probs[-1], iters[-1] = top.prob, top.iterations
    for k in range(nlev - 2, -1, -1):
        bound = upsample_linear(probs[k + 1], vols[k].shape)
        if skip_eps is not None:
            bid, _ = brick_ids(vols[k].shape, brick)
            keep = ~decided_bricks(bound, seed_levels[k], brick, skip_eps)[bid]
            res = solve_level(vols[k], seed_levels[k], brick, bound, params, solve_mask=keep)
        elif threads == 1:
            res = solve_level(vols[k], seed_levels[k], brick, bound, params)
        else:
            res = solve_level_threaded(vols[k], seed_levels[k], brick, bound, params, threads)
        probs[k], iters[k] = res.prob, res.iterations
    return HierarchyResult(probs, seed_levels, vols, iters, labels_from_prob(probs[0]))
