"""Multi-GPU execution: every level is split into z-slabs of brick rows across ranks.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  SURVEY.md §8(e): given level
k+1, the bricks of level k are independent Dirichlet problems (oracle/rw.py), so no collective
runs inside a solve; data moves only between levels, and only the planes a rank does not hold:

* **inputs and the LOD pyramid are slab-local.**  Rank r holds the level-0 planes of its share
  of the level-0 brick rows (its *LOD slab*); level k+1 of its slab is `lod_down` of its level-k
  slab plus two halo planes on either side (the [.25,.5,.25] conv reads one neighbour plane and
  the 2x mean pairs planes from an even start), so every coarse plane is computed by exactly one
  rank, bit-identical to the whole-volume pyramid.  Seed projection needs no halo.
* **the coarsest level is replicated**: its slabs are all-gathered (8 MB at config 4) and every
  rank solves it whole — the multigrid solve is deterministic, so the replicas agree bit for bit.
* **solve slabs follow the work.**  Before level k is solved, every rank scores the level-k brick
  rows by the undecided voxels (1e-3 < p < 1 - 1e-3) of the parent planes they read, plus a
  floor per voxel (decided bricks converge in a few iterations); the per-plane profile is
  all-reduced and every rank cuts the same contiguous split with equal score per rank.  The
  level's intensities / seeds (solve slab + one Dirichlet halo plane) and the parent solution
  planes its prolongation taps read are then redistributed point to point from whoever holds
  them (`batch_isend_irecv`; NCCL moves device tensors over NVLink, contiguous z-slices).
* **memory is slab-sized**: every per-level array a rank allocates covers its planes plus halo,
  never the whole level (except the replicated coarsest level).  The two-phase slab pipeline
  (slab c+1's brick systems built while slab c solves) runs inside each rank's slab.
* **per-level statistics are all-reduced** (counts summed; iteration maxima and solve times max).

Level-0 probabilities and labels stay distributed: rank r's result holds its solve slab
(`ShardResult.z0, z1`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

from .config import RWConfig


def level_shapes(shape, levels):
    out = [tuple(int(s) for s in shape)]
    for _ in range(levels - 1):
        out.append(tuple(-(-s // 2) for s in out[-1]))
    return out


def split_rows(n_rows: int, world: int):
    """Contiguous, balanced split of n_rows brick rows into `world` ranges."""
    return [(r * n_rows // world, (r + 1) * n_rows // world) for r in range(world)]


def split_by_weight(weights, world: int):
    """Contiguous split of rows with the given (non-negative) weights into `world` ranges of
    near-equal total weight: rank r takes the rows whose weight prefix midpoint falls into
    [r/world, (r+1)/world) of the total.  Deterministic (identical on every rank)."""
    n = len(weights)
    total = float(sum(weights))
    if n == 0:
        return [(0, 0)] * world
    if total <= 0:
        return split_rows(n, world)
    bounds = [0]
    acc = 0.0
    r = 1
    for j, w in enumerate(weights):
        mid = acc + 0.5 * w
        while r < world and mid >= total * r / world:
            bounds.append(j)
            r += 1
        acc += w
    while len(bounds) < world:
        bounds.append(n)
    bounds.append(n)
    return [(bounds[i], bounds[i + 1]) for i in range(world)]


def parent_planes(z0: int, z1: int, n_parent: int):
    """Parent planes [p0, p1) the prolongation reads for fine planes [z0, z1).

    Fine plane g reads parent planes (g/2 - 1, g/2) for even g and
    ((g-1)/2, (g+1)/2) for odd g, clamped (oracle/rw.py: upsample_linear).
    """
    def taps(g):
        j = g // 2
        return (max(j - 1, 0), j) if g % 2 == 0 else (j, min(j + 1, n_parent - 1))

    lo = min(taps(g)[0] for g in (z0, min(z0 + 1, z1 - 1)))
    hi = max(taps(g)[1] for g in (max(z1 - 2, z0), z1 - 1))
    return max(lo, 0), min(hi + 1, n_parent)


def rows_to_planes(rows, brick_z: int, nz: int):
    return [(min(a * brick_z, nz), min(b * brick_z, nz)) for a, b in rows]


@dataclass
class ShardPlan:
    """The static part of the split: level shapes and every rank's LOD slab per level."""
    shape: tuple
    brick: tuple
    levels: int
    rank: int
    world: int
    shapes: list = field(default_factory=list)
    lod: list = field(default_factory=list)  # per level: per rank (z0, z1) planes of its LOD slab

    @classmethod
    def build(cls, shape, brick, levels, rank, world, device=None):
        plan = cls(tuple(int(s) for s in shape), tuple(int(b) for b in brick), int(levels), rank, world)
        plan.shapes = level_shapes(shape, levels)
        n0 = plan.shapes[0][0]
        rows0 = -(-n0 // plan.brick[0])
        planes = rows_to_planes(split_rows(rows0, world), plan.brick[0], n0)
        plan.lod.append(planes)
        for k in range(1, levels):
            nk = plan.shapes[k][0]
            # brick[0] is even, so every slab starts on an even plane: coarse plane j belongs to
            # the rank holding fine plane 2j
            planes = [(min(-(-a // 2), nk), min(-(-b // 2), nk)) for a, b in planes]
            plan.lod.append(planes)
        return plan

    def lod_slab(self, level: int, rank: int | None = None):
        return self.lod[level][self.rank if rank is None else rank]


def halo(z0: int, z1: int, n: int, r: int):
    """[z0 - r, z1 + r) clipped to [0, n); empty ranges stay empty."""
    if z1 <= z0:
        return (z0, z0)
    return (max(z0 - r, 0), min(z1 + r, n))


def messages(have, need):
    """(src, dst, a, b): planes [a, b) to send from rank src to rank dst so that every rank ends up
    with its `need` range.  A rank never receives what it holds itself; every other needed plane
    comes from exactly one holder (the lowest rank), so replicated ranges are not sent twice."""
    out = []
    for dst, (n0, n1) in enumerate(need):
        todo = [(n0, n1)] if n1 > n0 else []
        h0, h1 = have[dst]
        if h1 > h0:  # own planes: a local copy
            todo = [seg for a, b in todo for seg in ((a, min(b, h0)), (max(a, h1), b)) if seg[1] > seg[0]]
        for src, (h0, h1) in enumerate(have):
            if src == dst or h1 <= h0 or not todo:
                continue
            rest = []
            for a, b in todo:
                c, d = max(a, h0), min(b, h1)
                if c < d:
                    out.append((src, dst, c, d))
                    rest += [seg for seg in ((a, c), (d, b)) if seg[1] > seg[0]]
                else:
                    rest.append((a, b))
            todo = rest
    return out


def redistribute(local: torch.Tensor, have, need, rank: int, group=None, shape_tail=None, dtype=None):
    """Planes [need[rank]) of a z-split level array, assembled from the ranks holding them.

    `local` holds this rank's planes [have[rank]); every rank calls this with the same `have` and
    `need` tables.  Own planes are copied locally; the others arrive point to point (NCCL: device
    tensors over NVLink; a non-NCCL backend with CUDA tensors stages through host memory).
    Planes nobody holds are left uninitialised (callers never read them)."""
    import torch.distributed as dist

    n0, n1 = need[rank]
    h0, h1 = have[rank]
    tail = tuple(local.shape[1:]) if shape_tail is None else tuple(shape_tail)
    dev = local.device
    out = torch.empty((max(n1 - n0, 0),) + tail, dtype=local.dtype if dtype is None else dtype, device=dev)
    a, b = max(n0, h0), min(n1, h1)
    if a < b:
        out[a - n0:b - n0].copy_(local[a - h0:b - h0])
    msgs = messages(have, need)
    if not msgs or not (dist.is_available() and dist.is_initialized()):
        return out
    stage = dev.type == "cuda" and dist.get_backend(group) != "nccl"
    ops, recvs = [], []
    for src, dst, a, b in msgs:
        if src == rank:
            t = local[a - h0:b - h0].contiguous()
            ops.append(dist.P2POp(dist.isend, t.cpu() if stage else t, dst, group=group))
        elif dst == rank:
            buf = torch.empty((b - a,) + tail, dtype=out.dtype, device="cpu" if stage else dev)
            ops.append(dist.P2POp(dist.irecv, buf, src, group=group))
            recvs.append((buf, a, b))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for buf, a, b in recvs:
        out[a - n0:b - n0].copy_(buf)
    return out


def _all_reduce(t: torch.Tensor, op, group=None) -> torch.Tensor:
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return t
    if t.is_cuda and dist.get_backend(group) != "nccl":
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        return h.to(t.device)
    dist.all_reduce(t, op=op, group=group)
    return t


def row_weights(parent_profile, n_fine: int, brick_z: int, plane_voxels_parent: int, floor: float = 0.05):
    """Score of each level-k brick row from the parent's undecided voxels per plane: the parent
    planes a row's prolongation reads, plus `floor` x their voxel count."""
    rows = -(-n_fine // brick_z)
    n_parent = len(parent_profile)
    w = []
    for j in range(rows):
        p0, p1 = parent_planes(j * brick_z, min((j + 1) * brick_z, n_fine), n_parent)
        w.append(float(sum(parent_profile[p0:p1])) + floor * plane_voxels_parent * (p1 - p0))
    return w


@dataclass
class ShardResult:
    prob: torch.Tensor            # level-0 probabilities of planes [z0, z1)
    labels: torch.Tensor | None   # level-0 labels of planes [z0, z1)
    z0: int
    z1: int
    stats: list                   # per level (level 0 first), all-reduced over ranks
    solve_rows: list              # per level < L-1: per rank (row0, row1) brick rows solved
    levels: list = field(default_factory=list)  # per level: (z0, z1, prob planes) this rank holds


def _merge(parts):
    from .device import _merge_stats, _resolve

    if isinstance(parts, list):
        return _merge_stats(parts) if parts else None
    return _resolve(parts)


def _reduce_stats(stats, device, group=None):
    import torch.distributed as dist

    keys_sum = ("bricks", "converged", "not_converged", "zero_rhs", "iterations_sum", "unknowns",
                "unknown_iterations")
    keys_max = ("iterations_max", "sweeps", "cg_ms", "path")
    n = len(stats)
    s = torch.zeros((n, len(keys_sum)), dtype=torch.float64, device=device)
    m = torch.full((n, len(keys_max)), -1.0, dtype=torch.float64, device=device)
    for k, st in enumerate(stats):
        if st is None:
            continue
        s[k] = torch.tensor([float(st[x]) for x in keys_sum], dtype=torch.float64)
        m[k] = torch.tensor([float(st[x]) for x in keys_max], dtype=torch.float64)
    s = _all_reduce(s, dist.ReduceOp.SUM, group)
    m = _all_reduce(m, dist.ReduceOp.MAX, group)
    out = []
    for k in range(n):
        d = {x: int(round(float(v))) for x, v in zip(keys_sum, s[k].tolist())}
        for x, v in zip(keys_max, m[k].tolist()):
            d[x] = float(v) if x == "cg_ms" else int(v)
        out.append(d)
    return out


def hierarchical_random_walker_sharded(vol_slab: torch.Tensor, seeds_slab: torch.Tensor, plan: ShardPlan,
                                       cfg: RWConfig = RWConfig(), *, workspace=None, want_labels: bool = True,
                                       group=None, level0_chunks: int | None = None, balance: bool = True,
                                       keep_levels: bool = False) -> ShardResult:
    """This rank's part of the hierarchical random walker.

    `vol_slab` / `seeds_slab`: the level-0 planes of this rank's LOD slab
    (`plan.lod_slab(0)`).  Every rank must call this with the same plan geometry."""
    import torch.distributed as dist

    from . import device

    rank, world, L = plan.rank, plan.world, plan.levels
    brick, shapes = plan.brick, plan.shapes
    bz = brick[0]
    dev = vol_slab.device
    workspace = workspace or device.Workspace(dev)
    if tuple(vol_slab.shape) != (plan.lod_slab(0)[1] - plan.lod_slab(0)[0],) + shapes[0][1:]:
        raise ValueError("vol_slab does not match this rank's level-0 LOD slab")

    # ---- LOD pyramid and seed levels of the slab.  Coarse plane j pairs fine planes 2j, 2j+1 and the
    # conv reads one more on either side: rank r's coarse planes [c0, c1) come from the fine window
    # [2 c0 - 2, 2 c1 + 2) (even start), the seeds from [2 c0, 2 c1)
    vols, seeds = [vol_slab], [seeds_slab]
    for k in range(L - 1):
        nk = shapes[k][0]
        have = plan.lod[k]
        coarse = plan.lod[k + 1]
        vneed = [(max(2 * c0 - 2, 0), min(2 * c1 + 2, nk)) if c1 > c0 else (2 * c0, 2 * c0) for c0, c1 in coarse]
        sneed = [(2 * c0, min(2 * c1, nk)) for c0, c1 in coarse]
        vwin = redistribute(vols[k], have, vneed, rank, group)
        swin = redistribute(seeds[k], have, sneed, rank, group)
        c0, c1 = coarse[rank]
        if c1 > c0:
            off = vneed[rank][0] // 2
            vols.append(device.lod_down(vwin)[c0 - off:c1 - off].contiguous())
            seeds.append(device.project_seeds(swin))
        else:
            vols.append(torch.empty((0,) + shapes[k + 1][1:], dtype=torch.float32, device=dev))
            seeds.append(torch.empty((0,) + shapes[k + 1][1:], dtype=torch.uint8, device=dev))
        del vwin, swin

    # ---- coarsest level: all-gathered, solved whole on every rank (deterministic replicas)
    top = L - 1
    full = [(0, shapes[top][0])] * world
    vtop = redistribute(vols[top], plan.lod[top], full, rank, group)
    stop = redistribute(seeds[top], plan.lod[top], full, rank, group)
    lab_top = torch.empty(shapes[top], dtype=torch.uint8, device=dev) if (want_labels and top == 0) else None
    ptop, st_top = device.solve_level(vtop, stop, shapes[top], None, cfg, labels_out=lab_top, workspace=workspace,
                                      stats_on_device=True)
    stats = [None] * L
    stats[top] = st_top
    parent, parent_have, replicated = ptop, full, True  # parent solution planes held by each rank
    solve_rows = [None] * L
    levels_kept = [(0, shapes[top][0], ptop)] if keep_levels else []
    res_prob, res_lab, res_z = ptop, lab_top, (0, shapes[top][0])

    for k in range(top - 1, -1, -1):
        nz = shapes[k][0]
        nrows = -(-nz // bz)
        # work-balanced contiguous split of the level's brick rows
        if balance:
            n_par = shapes[k + 1][0]
            prof = torch.zeros(n_par, dtype=torch.float64, device=dev)
            p0, p1 = parent_have[rank]
            if p1 > p0:
                und = ((parent > 1e-3) & (parent < 1 - 1e-3)).reshape(p1 - p0, -1).sum(1).to(torch.float64)
                prof[p0:p1] = und
            if not replicated:  # distributed parent: combine the slabs' profiles
                prof = _all_reduce(prof, dist.ReduceOp.SUM, group)
            weights = row_weights(prof.tolist(), nz, bz, math.prod(shapes[k + 1][1:]))
            rows = split_by_weight(weights, world)
        else:
            rows = split_rows(nrows, world)
        solve_rows[k] = rows
        planes = rows_to_planes(rows, bz, nz)
        z0, z1 = planes[rank]
        need = [halo(a, b, nz, 1) for a, b in planes]  # + the Dirichlet halo plane per side
        v_loc = redistribute(vols[k], plan.lod[k], need, rank, group)
        s_loc = redistribute(seeds[k], plan.lod[k], need, rank, group)
        # parent planes the prolongation of this rank's local planes reads
        pneed = [parent_planes(a, b, shapes[k + 1][0]) if b > a else (0, 0) for a, b in need]
        par = redistribute(parent, parent_have, pneed, rank, group)
        l0 = need[rank][0]
        lab = None
        if z1 > z0:
            lab = torch.empty(v_loc.shape, dtype=torch.uint8, device=dev) if (want_labels and k == 0) else None
            nb0 = (rows[rank][1] - rows[rank][0]) * math.prod(device.brick_grid(shapes[k][1:], brick[1:]))
            if k == 0 and level0_chunks is not None:
                chunks = level0_chunks
            else:  # as the single-GPU path: slab pipeline on large brick-resident levels
                chunks = 8 if nb0 >= 16384 else (2 if nb0 >= 4096 else 1)
            prob, parts = device._solve_level_chunked(
                v_loc, s_loc, brick, par, cfg, lab, workspace, chunks, None, z0=l0, fine_shape=shapes[k],
                parent_z0=pneed[rank][0], origin_z=z0 - l0, n_rows=rows[rank][1] - rows[rank][0])
            stats[k] = parts
            mine = prob[z0 - l0:z1 - l0]
        else:
            mine = torch.empty((0,) + shapes[k][1:], dtype=torch.float32, device=dev)
            stats[k] = []
        if keep_levels:
            levels_kept.append((z0, z1, mine))
        parent, parent_have, replicated = mine, planes, False
        res_prob, res_z = mine, (z0, z1)
        res_lab = lab[z0 - l0:z1 - l0] if lab is not None else None
        del v_loc, s_loc, par
    if dev.type == "cuda":
        torch.cuda.current_stream(dev).synchronize()
    local = [_merge(s) if s is not None else None for s in stats]
    merged = _reduce_stats(local, dev, group)
    return ShardResult(res_prob, res_lab, res_z[0], res_z[1], merged, solve_rows, levels_kept[::-1])
