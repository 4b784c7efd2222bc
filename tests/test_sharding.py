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


# -- the sharded hierarchical driver end to end, world_size 2 over gloo -------------------
# The level operators are swapped for the float64 oracle on CPU tensors, so the
# test exercises exactly the host logic that runs on GPUs: the shard plan, the
# per-level brick lists, and the point-to-point halo exchange of parent planes.

def _install_oracle_backend():
    from oracle import lod as olod
    from paper_2509_26213_b200 import device

    def lod_down(level):
        return torch.from_numpy(olod.lod_down(level.numpy()))

    def project_seeds(seeds):
        return torch.from_numpy(orw.project_seeds(seeds.numpy()))

    def upsample(parent, fine_shape, out=None):
        return torch.from_numpy(orw.upsample_linear(parent.numpy(), tuple(fine_shape)).astype(np.float32))

    def solve_level(vol, seeds, brick, bound, cfg, *, brick_list=None, out=None, labels_out=None,
                    workspace=None, origin=None, **_unused):
        params = orw.RWParams(beta=cfg.beta, min_weight=cfg.min_weight, tol=1e-10)
        b = None if bound is None else bound.numpy().astype(np.float64)
        res = orw.solve_level(vol.numpy(), seeds.numpy(), brick, b, params).prob.astype(np.float32)
        if out is None:
            out = torch.full(vol.shape, float("nan"))
        if brick_list is None:
            out.copy_(torch.from_numpy(res))
        else:
            bid, _ = orw.brick_ids(tuple(vol.shape), brick)
            sel = torch.from_numpy(np.isin(bid, brick_list.numpy()))
            out[sel] = torch.from_numpy(res)[sel]
        if labels_out is not None:
            labels_out.copy_(out > 0.5)
        return out, {"bricks": 0, "cg_ms": 0.0, "iterations_sum": 0}

    def upsample_window(parent, fine_shape, z0, z1, out):
        full = torch.from_numpy(orw.upsample_linear(parent.numpy(), tuple(fine_shape)).astype(np.float32))
        out.fill_(float("nan"))  # planes outside the window must never be read
        out[z0:z1] = full[z0:z1]
        return out

    device.lod_down = lod_down
    device.project_seeds = project_seeds
    device.upsample = upsample
    device.upsample_window = upsample_window
    device.solve_level = solve_level


def _sharded_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _install_oracle_backend()
        from paper_2509_26213_b200 import synthetic
        from paper_2509_26213_b200.config import RWConfig

        shape, brick, levels = (48, 16, 16), (8, 8, 8), 3
        vol = synthetic.phantom(shape)
        sd = synthetic.seeds(shape, "S1")
        plan = sharding.ShardPlan.build(shape, brick, levels, rank, world)
        for s in plan.shards:
            if s is not None:
                s.brick_list = torch.tensor(s.bricks[rank], dtype=torch.int32)
        res = sharding.hierarchical_random_walker_sharded(torch.from_numpy(vol), torch.from_numpy(sd), plan,
                                                          RWConfig(), want_labels=False)
        z0, z1 = plan.owned_planes(0, rank)
        q.put((rank, z0, z1, res.prob[z0:z1].numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_hierarchy_matches_single_process_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    from paper_2509_26213_b200 import synthetic

    shape = (48, 16, 16)
    vol = synthetic.phantom(shape)
    sd = synthetic.seeds(shape, "S1")
    ref = orw.hierarchical_random_walker(vol, sd, (8, 8, 8), 3, orw.RWParams(tol=1e-10)).prob[0].astype(np.float32)
    covered = np.zeros(shape[0], bool)
    for rank, z0, z1, part in got:
        assert not np.isnan(part).any()
        np.testing.assert_array_equal(part, ref[z0:z1])
        covered[z0:z1] = True
    assert covered.all()
