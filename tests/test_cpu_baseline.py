"""The extrapolated CPU baseline (oracle/cpu_baseline.py) on small cases: the
threaded whole-level solve equals the serial oracle, the LOD / seed helpers are bit-identical, the
brick chains solve real bricks from their true parents, and every level is accounted."""

from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import cpu_baseline as cb
from oracle import lod as olod
from oracle import rw as orw
from paper_2509_26213_b200 import synthetic


def test_threaded_helpers_match_the_serial_oracle():
    vol = synthetic.phantom((40, 36, 28))
    seeds = synthetic.seeds(vol.shape, "S2")
    with ThreadPoolExecutor(4) as pool:
        np.testing.assert_array_equal(cb.lod_down_threaded(vol, pool, 4), olod.lod_down(vol))
        np.testing.assert_array_equal(cb.project_seeds_threaded(seeds, pool, 4), orw.project_seeds(seeds))
        p = orw.RWParams(tol=1e-10)
        got, it = cb.solve_whole_threaded(vol, seeds, p, pool, 4)
        ref = orw.solve_level(vol, seeds, vol.shape, None, p)
        assert np.abs(got - ref.prob).max() < 1e-9 and abs(it - int(ref.iterations[0])) <= 2


def test_chain_blocks_equal_the_full_level_solve():
    """A chain's level-0 block, solved from the block one level up, is the full hierarchy's
    level 0 there (the prolongation taps of the interior children lie in the solved block)."""
    shape, brick, levels = (64, 64, 64), (8, 8, 8), 3
    vol = synthetic.phantom(shape)
    seeds = synthetic.seeds(shape, "S1")
    p = orw.RWParams(tol=1e-10)
    full = orw.hierarchical_random_walker(vol, seeds, brick, levels, p)
    vols, sds = full.volumes, full.seeds
    start = (1, 1, 1)  # level-1 block of 2x2x2 bricks at brick (1, 1, 1)
    lo1 = [s * b for s, b in zip(start, brick)]
    blk1 = cb._block_solve(vols[1], sds[1], full.prob[2], (0, 0, 0), vols[1].shape, brick, lo1,
                           [a + 2 * b for a, b in zip(lo1, brick)], p)
    np.testing.assert_allclose(blk1, full.prob[1][tuple(slice(a, a + 2 * b) for a, b in zip(lo1, brick))],
                               atol=1e-9)
    lo0 = [(2 * s + 1) * b for s, b in zip(start, brick)]
    blk0 = cb._block_solve(vols[0], sds[0], blk1, tuple(lo1), vols[0].shape, brick, lo0,
                           [a + 2 * b for a, b in zip(lo0, brick)], p)
    np.testing.assert_allclose(blk0, full.prob[0][tuple(slice(a, a + 2 * b) for a, b in zip(lo0, brick))],
                               atol=1e-9)
    with pytest.raises(RuntimeError):  # a block whose taps leave the parent window
        cb._block_solve(vols[0], sds[0], blk1, tuple(lo1), vols[0].shape, brick, [0, 0, 0], [16, 16, 16], p)


def test_step_accounts_every_level():
    vol = synthetic.phantom((64, 64, 64))
    seeds = synthetic.seeds(vol.shape, "S1")
    base = cb.C4Baseline(vol, seeds, (16, 16, 16), 3, orw.RWParams(tol=1e-6), cores=2, chains=2, slab_planes=16)
    try:
        total, parts = base.step()
    finally:
        base.close()
    assert set(parts) == {"lod_and_seeds", "coarsest", "prolongation", "level1_bricks", "level0_bricks"}
    assert all(v > 0 for v in parts.values()) and abs(total - sum(parts.values())) < 1e-9
    assert base.top_iterations > 0 and base.top_full_seconds > 0
