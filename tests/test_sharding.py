"""Host-side multi-GPU logic on CPU: the slab plan, work-balanced splits, plane redistribution
and the whole sharded hierarchy over world_size-2 / 3 gloo process groups (the level operators
swapped for the float64 oracle on CPU tensors, so exactly the host logic that runs on GPUs is
exercised: LOD slabs with halos, the all-gathered coarsest level, the per-level splits, the
point-to-point redistribution of volumes, seeds and parent planes, the stats reduction)."""

import os
import random
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import rw as orw
from paper_2509_26213_b200 import sharding


def brute_parent_planes(z0, z1, n_parent):
    used = set()
    for g in range(z0, z1):
        j = g // 2
        taps = (max(j - 1, 0), j) if g % 2 == 0 else (j, min(j + 1, n_parent - 1))
        used.update(taps)
    return min(used), max(used) + 1


@pytest.mark.parametrize("n_fine", [1, 2, 7, 64, 65])
def test_parent_planes_match_taps(n_fine):
    n_parent = -(-n_fine // 2)
    for z0 in range(n_fine):
        for z1 in range(z0 + 1, n_fine + 1):
            assert sharding.parent_planes(z0, z1, n_parent) == brute_parent_planes(z0, z1, n_parent)


def test_parent_planes_agree_with_oracle_upsample():
    # perturbing a parent plane outside parent_planes() must not change the fine planes
    rng = np.random.default_rng(1)
    parent = rng.random((9, 3))
    fine_shape = (17, 5)
    z0, z1 = 6, 11
    p0, p1 = sharding.parent_planes(z0, z1, 9)
    base = orw.upsample_linear(parent, fine_shape)[z0:z1]
    pert = parent.copy()
    pert[:p0] += 100.0
    pert[p1:] += 100.0
    np.testing.assert_array_equal(orw.upsample_linear(pert, fine_shape)[z0:z1], base)


@pytest.mark.parametrize("world", [1, 2, 3, 8, 40])
def test_lod_slabs_partition_every_level(world):
    shape, brick, levels = (300, 40, 24), (32, 32, 32), 4
    plan = sharding.ShardPlan.build(shape, brick, levels, 0, world)
    for k, planes in enumerate(plan.lod):
        n = plan.shapes[k][0]
        cover = [z for a, b in planes for z in range(a, b)]
        assert cover == list(range(n))  # contiguous, disjoint, complete, in rank order
        if k > 0:  # coarse plane j lives with fine plane 2j
            for (a, b), (fa, fb) in zip(planes, plan.lod[k - 1]):
                assert all(fa <= 2 * j < fb for j in range(a, b))
    assert all(a % 32 == 0 for a, _ in plan.lod[0])


def test_split_by_weight_is_contiguous_and_balanced():
    rnd = random.Random(5)
    for _ in range(300):
        n, world = rnd.randint(1, 60), rnd.randint(1, 9)
        w = [rnd.choice([0.0, 0.1, 1.0, 5.0, 40.0]) * rnd.random() for _ in range(n)]
        parts = sharding.split_by_weight(w, world)
        assert len(parts) == world and parts[0][0] == 0 and parts[-1][1] == n
        assert all(a <= b for a, b in parts) and all(p[1] == q[0] for p, q in zip(parts, parts[1:]))
        total = sum(w)
        if total > 0:  # no rank exceeds its share by more than one row's weight
            assert max(sum(w[a:b]) for a, b in parts) <= total / world + max(w) + 1e-9
    # heavy rows in the middle pull the cuts towards them
    w = [1.0] * 16 + [100.0] * 4 + [1.0] * 16
    parts = sharding.split_by_weight(w, 4)
    assert [b - a for a, b in parts] != [9, 9, 9, 9] and all(sum(w[a:b]) <= 120 for a, b in parts)


def test_messages_cover_needs_once():
    rnd = random.Random(2)
    for _ in range(500):
        n, world = rnd.randint(1, 50), rnd.randint(1, 6)
        cuts = sorted(rnd.randint(0, n) for _ in range(world - 1))
        have = list(zip([0] + cuts, cuts + [n]))
        if rnd.random() < 0.2:  # replicated
            have = [(0, n)] * world
        need = []
        for _ in range(world):
            a = rnd.randint(0, n)
            need.append((a, rnd.randint(a, n)))
        got = {d: [] for d in range(world)}
        for src, dst, a, b in sharding.messages(have, need):
            assert src != dst and have[src][0] <= a < b <= have[src][1]
            got[dst].append((a, b))
        for d in range(world):
            planes = [z for a, b in got[d] for z in range(a, b)]
            own = set(range(*have[d]))
            assert len(planes) == len(set(planes)) and not (set(planes) & own)  # each plane once
            assert set(range(*need[d])) <= own | set(planes)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(target, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    return got


def _redistribute_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 23
        truth = torch.arange(n * 6, dtype=torch.float64).reshape(n, 2, 3)
        have = [(0, 9), (9, 9), (9, 23)][:world] if world == 3 else [(0, 12), (12, 23)]
        need = [(5, 23), (0, 23), (8, 10)][:world] if world == 3 else [(10, 23), (0, 14)]
        a, b = have[rank]
        out = sharding.redistribute(truth[a:b].clone(), have, need, rank)
        c, d = need[rank]
        q.put((rank, bool(torch.equal(out, truth[c:d]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_redistribute_gloo(world):
    assert all(ok for _, ok in _spawn(_redistribute_worker, world))


# -- the sharded hierarchical driver end to end over gloo, oracle level operators ----------


def _install_oracle_backend():
    from oracle import lod as olod
    from paper_2509_26213_b200 import device

    zero = {k: 0 for k in ("bricks", "converged", "not_converged", "zero_rhs", "iterations_sum", "unknowns",
                           "unknown_iterations", "iterations_max", "sweeps", "path")}
    zero["cg_ms"] = 0.0

    def params(cfg):
        return orw.RWParams(beta=cfg.beta, min_weight=cfg.min_weight, tol=1e-10)

    def lod_down(level):
        return torch.from_numpy(olod.lod_down(level.numpy()))

    def project_seeds(seeds):
        return torch.from_numpy(orw.project_seeds(seeds.numpy()))

    def solve_level(vol, seeds, brick, bound, cfg, *, labels_out=None, **_unused):
        assert bound is None  # the sharded driver solves only the coarsest level whole
        res = orw.solve_level(vol.numpy(), seeds.numpy(), tuple(vol.shape), None, params(cfg))
        out = torch.from_numpy(res.prob)
        if labels_out is not None:
            labels_out.copy_(out > 0.5)
        return out, dict(zero, bricks=1)

    def chunked(vol, seeds, brick, parent, cfg, labels_out, workspace, chunks, on_chunk, *, z0, fine_shape,
                parent_z0, origin_z, n_rows):
        nz = vol.shape[0]
        # the bound from a NaN-padded parent: a tap outside the window the driver shipped
        # poisons the result
        pshape = tuple(-(-s // 2) for s in fine_shape)
        full = np.full(pshape, np.nan)
        full[parent_z0:parent_z0 + parent.shape[0]] = parent.numpy()
        lo = (z0,) + (0,) * (len(fine_shape) - 1)
        hi = (z0 + nz,) + tuple(fine_shape[1:])
        bound = orw.upsample_linear_window(full, tuple(fine_shape), lo, hi)
        mask = np.zeros(vol.shape, bool)
        mask[origin_z:min(origin_z + n_rows * brick[0], nz)] = True
        res = orw.solve_level(vol.numpy(), seeds.numpy(), brick, bound, params(cfg), solve_mask=mask,
                              origin=lo)
        out = torch.from_numpy(res.prob)
        if labels_out is not None:
            labels_out.copy_(out > 0.5)
        return out, [dict(zero, bricks=int(n_rows))]

    device.lod_down = lod_down
    device.project_seeds = project_seeds
    device.solve_level = solve_level
    device._solve_level_chunked = chunked


CASES = {"even": ((80, 16, 16), (8, 8, 8), 3), "ragged": ((75, 12, 10), (8, 8, 8), 3),
         "2d": ((70, 22), (8, 8), 3)}


def _sharded_worker(rank, world, port, q, case, balance):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _install_oracle_backend()
        from paper_2509_26213_b200 import synthetic
        from paper_2509_26213_b200.config import RWConfig

        shape, brick, levels = CASES[case]
        vol = synthetic.phantom(shape)
        sd = synthetic.seeds(shape, "S2")
        plan = sharding.ShardPlan.build(shape, brick, levels, rank, world)
        a, b = plan.lod_slab(0)
        res = sharding.hierarchical_random_walker_sharded(torch.from_numpy(vol[a:b].copy()),
                                                          torch.from_numpy(sd[a:b].copy()), plan, RWConfig(),
                                                          balance=balance)
        q.put((rank, res.z0, res.z1, res.prob.numpy(), res.labels.numpy(), res.stats, res.solve_rows))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world,balance", [("even", 2, True), ("ragged", 3, True), ("ragged", 2, False),
                                                ("2d", 2, True)])
def test_sharded_hierarchy_matches_single_process(case, world, balance):
    from paper_2509_26213_b200 import synthetic

    got = _spawn(_sharded_worker, world, case, balance)
    shape, brick, levels = CASES[case]
    vol = synthetic.phantom(shape)
    sd = synthetic.seeds(shape, "S2")
    ref = orw.hierarchical_random_walker(vol, sd, brick, levels, orw.RWParams(tol=1e-10))
    covered = np.zeros(shape[0], int)
    for rank, z0, z1, part, lab, stats, rows in got:
        assert not np.isnan(part).any()
        np.testing.assert_array_equal(part, ref.prob[0][z0:z1])
        np.testing.assert_array_equal(lab, ref.labels[z0:z1])
        covered[z0:z1] += 1
        # every rank holds the same all-reduced stats and the same splits
        assert stats == got[0][5] and rows == got[0][6]
        assert stats[-1]["bricks"] == world  # the replicated coarsest solve, counted per rank
        grid0 = -(-shape[0] // brick[0])
        assert stats[0]["bricks"] == grid0 and rows[0][-1][1] == grid0
    assert (covered == 1).all()


def test_roi_brick_boxes_cover_the_prolongation_taps():
    """Every parent voxel the listed bricks (+1 halo) of level k read is inside level k+1's box."""
    from paper_2509_26213_b200 import device

    rnd = random.Random(9)
    for _ in range(200):
        nd = rnd.choice([2, 3])
        brick = tuple(rnd.choice([8, 16]) for _ in range(nd))
        shape0 = tuple(rnd.randint(20, 120) for _ in range(nd))
        shapes = sharding.level_shapes(shape0, rnd.randint(2, 4))
        lo = [rnd.randint(0, n - 1) for n in shape0]
        hi = [rnd.randint(a + 1, n) for a, n in zip(lo, shape0)]
        boxes = device.roi_brick_boxes(shapes, brick, (lo, hi))
        assert boxes[-1] is None and len(boxes) == len(shapes)
        b0, b1 = boxes[0]
        assert all(x * b <= a and y * b >= h for x, y, a, h, b in zip(b0, b1, lo, hi, brick))
        for k in range(len(shapes) - 2):
            (b0, b1), (p0, p1) = boxes[k], boxes[k + 1]
            for d in range(nd):
                v0, v1 = max(b0[d] * brick[d] - 1, 0), min(b1[d] * brick[d] + 1, shapes[k][d])
                t0, t1 = brute_parent_planes(v0, v1, shapes[k + 1][d])
                assert p0[d] * brick[d] <= t0 and min(p1[d] * brick[d], shapes[k + 1][d]) >= t1
