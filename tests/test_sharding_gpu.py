"""The sharded multi-rank path on real kernels: 2 ranks share cuda:0 (gloo
transport, planes staged through the host; NCCL needs one GPU per rank and the
GPU box has one).  The ranks' kernels never wait on each other — the halo
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


CASES = {"resident": ((128, 64, 64), (32, 32, 32), 3), "streaming": ((96, 40, 40), (16, 16, 16), 3)}


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_26213_b200 import sharding, synthetic
        from paper_2509_26213_b200.config import RWConfig

        shape, brick, levels = CASES[case]
        dev = torch.device("cuda", 0)
        vol = torch.from_numpy(synthetic.phantom(shape)).to(dev)
        sd = torch.from_numpy(synthetic.seeds(shape, "S1")).to(dev)
        plan = sharding.ShardPlan.build(shape, brick, levels, rank, world, device=dev)
        res = sharding.hierarchical_random_walker_sharded(vol, sd, plan, RWConfig(tol=1e-7))
        torch.cuda.synchronize()
        z0, z1 = plan.owned_planes(0, rank)
        q.put((rank, z0, z1, res.prob[z0:z1].cpu().numpy(), res.labels[z0:z1].cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", sorted(CASES))
def test_two_ranks_on_one_gpu_match_single_process(case):
    from paper_2509_26213_b200 import device, synthetic
    from paper_2509_26213_b200.config import RWConfig

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
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
    covered = np.zeros(shape[0], bool)
    for rank, z0, z1, p, lab in got:
        np.testing.assert_array_equal(p, p_ref[z0:z1])
        np.testing.assert_array_equal(lab, l_ref[z0:z1])
        covered[z0:z1] = True
    assert covered.all()
