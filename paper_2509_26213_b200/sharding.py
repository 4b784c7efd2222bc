"""Multi-GPU execution: bricks of every level sharded across ranks.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  Given
level k+1, the bricks of level k are independent Dirichlet problems
(oracle/rw.py), so level k is split into contiguous z-slabs of brick rows,
one per rank, and solved with the `brick_list` argument of the level solver
— no collective inside a solve.  The coarsest level (one brick) is solved
redundantly on every rank; it is deterministic, so all replicas agree
bit for bit.

The only data exchange is the inter-level halo: before level k is
upsampled for level k-1, every rank needs the parent planes its level-(k-1)
bricks (plus their one-voxel Dirichlet halo) read through the multilinear
prolongation taps.  The planes it does not own itself are received from
their owners with point-to-point sends/receives (`batch_isend_irecv`; on
NCCL they run over NVLink).  Level slabs are contiguous in the z-major HBM
layout, so each message is one contiguous slice.

The LOD pyramid and seed projections are computed on every rank from the
resident full-resolution input (a few ms of HBM streaming at 1024^3,
SURVEY.md §8(e)); level-0 probabilities/labels stay distributed (each rank's
output is valid inside its own slab).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .config import RWConfig

CG_BYTES_PER_VOXEL_ITER = {2: 48, 3: 52}


def cg_bytes_per_voxel_iter(ndim: int) -> int:
    """Algorithmic HBM bytes per brick voxel per CG iteration (csrc/rwb_solve.cu header)."""
    return CG_BYTES_PER_VOXEL_ITER[ndim]


def level_shapes(shape, levels):
    out = [tuple(int(s) for s in shape)]
    for _ in range(levels - 1):
        out.append(tuple(-(-s // 2) for s in out[-1]))
    return out


def split_rows(n_rows: int, world: int):
    """Contiguous, balanced split of n_rows brick rows into `world` ranges."""
    return [(r * n_rows // world, (r + 1) * n_rows // world) for r in range(world)]


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


@dataclass
class LevelShard:
    shape: tuple
    rows: list                      # per rank: owned brick rows [r0, r1) along dim 0
    planes: list                    # per rank: owned planes [z0, z1) along dim 0
    bricks: list                    # per rank: owned brick indices (row-major)
    brick_list: torch.Tensor | None = None  # this rank's bricks, int32 on device


@dataclass
class ShardPlan:
    shape: tuple
    brick: tuple
    levels: int
    rank: int
    world: int
    shards: list = field(default_factory=list)  # per level (coarsest: None = replicated)

    @classmethod
    def build(cls, shape, brick, levels, rank, world, device=None):
        shapes = level_shapes(shape, levels)
        plan = cls(tuple(shape), tuple(brick), levels, rank, world)
        for k, s in enumerate(shapes):
            if k == levels - 1:
                plan.shards.append(None)
                continue
            grid = [-(-a // b) for a, b in zip(s, brick)]
            rows = split_rows(grid[0], world)
            per_row = 1
            for g in grid[1:]:
                per_row *= g
            planes = [(min(r0 * brick[0], s[0]), min(r1 * brick[0], s[0])) for r0, r1 in rows]
            bricks = [list(range(r0 * per_row, r1 * per_row)) for r0, r1 in rows]
            shard = LevelShard(s, rows, planes, bricks)
            if device is not None:
                shard.brick_list = torch.tensor(bricks[rank], dtype=torch.int32, device=device)
            plan.shards.append(shard)
        return plan

    def owned_planes(self, level: int, rank: int):
        """Planes of `level` that `rank` holds valid after solving it."""
        if level == self.levels - 1:
            return (0, level_shapes(self.shape, self.levels)[level][0])
        return self.shards[level].planes[rank]

    def needed_planes(self, level: int, rank: int):
        """Planes of `level` rank needs to upsample level-1 (rank's own bricks + halo)."""
        shapes = level_shapes(self.shape, self.levels)
        child = level - 1
        z0, z1 = self.shards[child].planes[rank]
        if z1 <= z0:
            return (0, 0)
        return parent_planes(max(z0 - 1, 0), min(z1 + 1, shapes[child][0]), shapes[level][0])


def halo_messages(plan: ShardPlan, level: int):
    """(src, dst, z0, z1) plane ranges to move after `level` is solved."""
    msgs = []
    if level == plan.levels - 1:
        return msgs  # replicated coarsest level: everyone already has it
    for dst in range(plan.world):
        n0, n1 = plan.needed_planes(level, dst)
        for src in range(plan.world):
            if src == dst:
                continue
            o0, o1 = plan.owned_planes(level, src)
            a, b = max(n0, o0), min(n1, o1)
            if a < b:
                msgs.append((src, dst, a, b))
    return msgs


def exchange_halo(plan: ShardPlan, level: int, prob: torch.Tensor, group=None):
    """Receive the parent planes this rank needs from their owners (point to point).

    NCCL moves device tensors directly (NVLink); backends without device
    support for point-to-point (gloo: CPU tests, several ranks sharing one
    GPU in tests) get the planes staged through host memory.
    """
    import torch.distributed as dist

    msgs = halo_messages(plan, level)
    if not msgs:
        return
    stage = prob.is_cuda and dist.get_backend(group) != "nccl"
    sends, recvs = [], []
    for src, dst, a, b in msgs:
        if src == plan.rank:
            t = prob[a:b].contiguous()
            sends.append((t.cpu() if stage else t, dst))
        elif dst == plan.rank:
            buf = torch.empty(prob[a:b].shape, dtype=prob.dtype, device="cpu" if stage else prob.device)
            recvs.append((buf, src, a, b))
    ops = [dist.P2POp(dist.isend, t, dst, group=group) for t, dst in sends]
    ops += [dist.P2POp(dist.irecv, buf, src, group=group) for buf, src, _, _ in recvs]
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for buf, _, a, b in recvs:
        prob[a:b].copy_(buf)


def upsample_planes(plan: ShardPlan, level: int):
    """Planes of `level` (< L-1) this rank's bricks and their 1-voxel halo read."""
    z0, z1 = plan.shards[level].planes[plan.rank]
    if z1 <= z0:
        return (0, 0)
    return (max(z0 - 1, 0), min(z1 + 1, plan.shards[level].shape[0]))


def hierarchical_random_walker_sharded(volume, seeds, plan: ShardPlan, cfg: RWConfig = RWConfig(), *,
                                       workspace=None, want_labels=True, group=None):
    """`device.hierarchical_random_walker` with this rank's bricks only."""
    from . import device

    lists = [s.brick_list if s is not None else None for s in plan.shards]
    windows = [upsample_planes(plan, k) if k < plan.levels - 1 else None for k in range(plan.levels)]

    def exchange(level, prob):
        exchange_halo(plan, level, prob, group)

    return device.hierarchical_random_walker(volume, seeds, plan.brick, plan.levels, cfg, want_labels=want_labels,
                                             workspace=workspace, brick_lists=lists, exchange=exchange,
                                             upsample_planes=windows)
