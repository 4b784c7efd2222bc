"""Host-side multi-GPU logic on CPU: shard plans, halo planes, and the halo
exchange itself over a world_size-2 gloo process group."""

import os
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


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_partitions_every_level(world):
    shape, brick, levels = (256, 96, 80), (32, 32, 32), 3
    for rank in range(world):
        plan = sharding.ShardPlan.build(shape, brick, levels, rank, world)
        assert plan.shards[-1] is None
        for k, sh in enumerate(plan.shards[:-1]):
            grid = [-(-a // b) for a, b in zip(sh.shape, brick)]
            allb = sorted(b for r in range(world) for b in sh.bricks[r])
            assert allb == list(range(int(np.prod(grid))))
            planes = [p for r in range(world) for p in range(*sh.planes[r])]
            assert planes == list(range(sh.shape[0]))
            # bricks of a rank lie inside its planes
            bid, _ = orw.brick_ids(sh.shape, brick)
            z0, z1 = sh.planes[rank]
            owned = np.isin(bid, sh.bricks[rank])
            zz = np.nonzero(owned.any(axis=(1, 2)))[0]
            if len(zz):
                assert zz.min() >= z0 and zz.max() < z1


def test_halo_messages_cover_needs():
    plan = sharding.ShardPlan.build((128, 64, 64), (16, 16, 16), 3, 0, 4)
    for level in range(1, plan.levels):
        msgs = sharding.halo_messages(plan, level)
        for dst in range(plan.world):
            n0, n1 = plan.needed_planes(level, dst)
            have = set(range(*plan.owned_planes(level, dst)))
            for src, d, a, b in msgs:
                if d == dst:
                    assert src != dst
                    have.update(range(a, b))
            assert set(range(n0, n1)) <= have
    assert sharding.halo_messages(plan, plan.levels - 1) == []


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape, brick, levels = (64, 8, 8), (8, 8, 8), 3
        plan = sharding.ShardPlan.build(shape, brick, levels, rank, world)
        ok = True
        for level in range(1, levels - 1):
            n = sharding.level_shapes(shape, levels)[level]
            truth = torch.arange(int(np.prod(n)), dtype=torch.float32).reshape(n)
            prob = torch.full(n, float("nan"))
            o0, o1 = plan.owned_planes(level, rank)
            prob[o0:o1] = truth[o0:o1]
            sharding.exchange_halo(plan, level, prob)
            a, b = plan.needed_planes(level, rank)
            ok &= bool(torch.equal(prob[a:b], truth[a:b]))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    results = dict(q.get(timeout=5) for _ in procs)
    assert results == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)
