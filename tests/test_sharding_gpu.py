"""The sharded multi-rank path on real kernels: 2 or 3 ranks share cuda:0 (gloo
transport, planes staged through the host; NCCL needs one GPU per rank and the
GPU box has one).  Each rank starts from its own level-0 slab only.  The ranks' kernels never wait on each other — the halo
exchange is host-driven between levels — so sharing a GPU is safe.  Every
rank's slab must be bit-identical to the single-process solve."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {"resident": ((128, 64, 64), (32, 32, 32), 3), "streaming": ((96, 40, 40), (16, 16, 16), 3),
         "resident2d": ((448, 192), (64, 64), 3), "ragged": ((150, 70, 40), (32, 32, 32), 3)}


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_26213_b200 import sharding, synthetic
        from paper_2509_26213_b200.config import RWConfig

        shape, brick, levels = CASES[case]
        dev = torch.device("cuda", 0)
        plan = sharding.ShardPlan.build(shape, brick, levels, rank, world)
        a, b = plan.lod_slab(0)
        vol = torch.from_numpy(synthetic.phantom(shape)[a:b].copy()).to(dev)
        sd = torch.from_numpy(synthetic.seeds(shape, "S1")[a:b].copy()).to(dev)
        res = sharding.hierarchical_random_walker_sharded(vol, sd, plan, RWConfig(tol=1e-7))
        torch.cuda.synchronize()
        q.put((rank, res.z0, res.z1, res.prob.cpu().numpy(), res.labels.cpu().numpy(), res.stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("resident", 2), ("streaming", 2), ("resident2d", 2), ("ragged", 3)])
def test_ranks_on_one_gpu_match_single_process(case, world):
    from paper_2509_26213_b200 import device, synthetic
    from paper_2509_26213_b200.config import RWConfig

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    shape, brick, levels = CASES[case]
    ref = device.hierarchical_random_walker(torch.from_numpy(synthetic.phantom(shape)).cuda(),
                                            torch.from_numpy(synthetic.seeds(shape, "S1")).cuda(), brick, levels,
                                            RWConfig(tol=1e-7))
    torch.cuda.synchronize()
    p_ref, l_ref = ref.prob.cpu().numpy(), ref.labels.cpu().numpy()
    covered = np.zeros(shape[0], int)
    for rank, z0, z1, p, lab, stats in got:
        np.testing.assert_array_equal(p, p_ref[z0:z1])
        np.testing.assert_array_equal(lab, l_ref[z0:z1])
        covered[z0:z1] += 1
        assert stats == got[0][5]  # all-reduced: identical on every rank
        assert [s["bricks"] for s in stats[:-1]] == [st["bricks"] for st in ref.stats[:-1]]
        assert stats[0]["not_converged"] == 0
    assert (covered == 1).all()
