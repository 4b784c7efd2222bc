"""Operator mode: the librwb operators as drop-in `chunkcast` OperatorNodes.

CPU tests check graph structure (metadata, footprints, ids, errors) against
the reference package; GPU tests resolve the nodes through the reference's
own `Engine` and compare with the reference LOD, the device-batched path
and the oracle.  `chunkcast` comes from the environment or baseline/_ref.
"""

import numpy as np
import pytest

from conftest import load_golden, reference_package
from paper_2509_26213_b200 import ops as rwops
from paper_2509_26213_b200 import synthetic

cc = reference_package()  # fails (does not skip) when the reference is missing



def _engine():
    from chunkcast.engine import Engine, EngineConfig
    from chunkcast.store import StoreConfig

    return Engine(EngineConfig(stores=StoreConfig(ram_capacity=1 << 28), worker_pool_size=4))


def _dense(engine, node):
    out = np.zeros(node.md.element_type.payload_shape(node.md.size), dtype=node.md.element_type.np_dtype)
    positions = list(node.md.chunk_positions())
    for pos, arr in zip(positions, engine.resolve(node, positions)):
        b, e = node.md.chunk_logical_region(pos)
        out[tuple(slice(x, y) for x, y in zip(b, e))] = arr[tuple(slice(0, y - x) for x, y in zip(b, e))]
    return out


# -- structure (CPU) -----------------------------------------------------------------


def test_pyramid_metadata_matches_reference_build_lod():
    src = cc.ops.source_from_array(np.zeros((100, 70, 40), np.float32), (16, 16, 16),
                                   embedding=(0.5, 1.0, 2.0))
    ref = cc.ops.build_lod(src)
    ours = rwops.build_lod(src)
    assert ours.num_levels == ref.num_levels
    for k in range(ref.num_levels):
        assert ours.node(k).md == ref.node(k).md
        assert ours.embedding(k) == ref.embedding(k)


def test_level_cap():
    src = cc.ops.source_from_array(np.zeros((256, 256), np.float32), (32, 32))
    assert rwops.build_lod(src, levels=2).num_levels == 2
    with pytest.raises(cc.ops.OperatorError):
        rwops.build_lod(src, levels=9)


def test_random_walker_footprint_is_dilated_neighbourhood():
    # like the reference's conv footprint test (test_engine.py:62-81): 3^d chunks, clipped at corners
    shape, chunk = (128, 128, 128), (16, 16, 16)
    vol = cc.ops.source_from_array(np.zeros(shape, np.float32), chunk)
    seeds = cc.ops.source_from_array(np.zeros(shape, np.uint8), chunk)
    pyr = rwops.hierarchical_random_walker(vol, seeds, levels=2)
    fine = pyr.node(0)
    deps = fine.dependencies((3, 4, 2))
    assert len(deps[0]) == 27 and deps[0] == deps[1]
    assert len(fine.dependencies((0, 0, 0))[0]) == 8
    # parent footprint through the prolongation taps: fine [47,65)x[63,81)x[31,49)
    # -> parent rows [23,33)x[31,41)x[15,25) -> parent chunks {1,2}x{1,2}x{0,1}
    assert sorted(deps[2]) == sorted((a, b, c) for a in (1, 2) for b in (1, 2) for c in (0, 1))
    top = pyr.node(1)
    assert len(top.dependencies((0, 0, 0))[0]) == 64  # whole coarsest level


def test_ids_are_deterministic_and_parameter_sensitive():
    data = synthetic.phantom((32, 32))
    vol = cc.ops.source_from_array(data, (16, 16))
    seeds = cc.ops.source_from_array(synthetic.seeds((32, 32)), (16, 16))
    a = rwops.hierarchical_random_walker(vol, seeds).node(0)
    b = rwops.hierarchical_random_walker(vol, seeds).node(0)
    c = rwops.hierarchical_random_walker(vol, seeds, beta=50.0).node(0)
    assert a.op_id == b.op_id and a.op_id != c.op_id


def test_type_errors_raise_operator_error():
    f32 = cc.ops.source_from_array(np.zeros((8, 8), np.float32), (4, 4))
    u8 = cc.ops.source_from_array(np.zeros((8, 8), np.uint8), (4, 4))
    with pytest.raises(cc.ops.OperatorError):
        rwops.random_walker(u8, u8)
    with pytest.raises(cc.ops.OperatorError):
        rwops.random_walker(f32, f32)
    with pytest.raises(cc.ops.OperatorError):
        rwops.rw_weights(u8)
    with pytest.raises(cc.ops.OperatorError):
        rwops.downsample_mean(u8)
    with pytest.raises(cc.ops.OperatorError):
        rwops.downsample_mean(f32, dims=(2,))


def test_unsmoothed_pyramid_and_dims_metadata_match_reference():
    src = cc.ops.source_from_array(np.zeros((100, 70, 40), np.float32), (16, 16, 16), embedding=(0.5, 1.0, 2.0))
    ref = cc.ops.build_lod(src, smooth=False)
    ours = rwops.build_lod(src, smooth=False)
    assert ours.num_levels == ref.num_levels
    for k in range(ref.num_levels):
        assert ours.node(k).md == ref.node(k).md and ours.embedding(k) == ref.embedding(k)
    for dims in [(0,), (1, 2), None]:
        r, o = cc.ops.downsample_mean(src, dims), rwops.downsample_mean(src, dims)
        assert o.md == r.md and o.embedding == r.embedding
        assert o.dependencies((1, 1, 0)) == r.dependencies((1, 1, 0))


# -- through the reference Engine (GPU) ------------------------------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["r3d", "r2d", "phantom3d"])
def test_engine_resolves_lod_bit_exact(name):
    import json
    import os

    from conftest import GOLDEN

    meta = json.load(open(os.path.join(GOLDEN, "MANIFEST.json")))["lod"][name]
    g = load_golden("lod_reference.npz")
    x = synthetic.phantom(tuple(meta["shape"])) if name.startswith("phantom") else g[f"{name}/input"]
    pyr = rwops.build_lod(cc.ops.source_from_array(x, meta["chunk"]))
    assert pyr.num_levels == meta["levels"]
    with _engine() as eng:
        for k in range(1, pyr.num_levels):
            np.testing.assert_array_equal(_dense(eng, pyr.node(k)), g[f"{name}/level{k}"])


@pytest.mark.gpu
@pytest.mark.parametrize("shape,chunk", [((37, 50, 23), (16, 16, 16)), ((99, 70), (32, 16))])
def test_engine_unsmoothed_pyramid_and_dims_bit_exact(shape, chunk):
    """build_lod(smooth=False) and downsample_mean(dims=...) through the reference Engine equal the
    reference's own numpy operators resolved by the same Engine, byte for byte (ops.py:611-727)."""
    x = np.random.default_rng(7).normal(0.3, 0.2, shape).astype(np.float32)
    src = cc.ops.source_from_array(x, chunk)
    ref, ours = cc.ops.build_lod(src, smooth=False), rwops.build_lod(src, smooth=False)
    assert ours.num_levels == ref.num_levels > 1
    with _engine() as eng:
        for k in range(1, ref.num_levels):
            np.testing.assert_array_equal(_dense(eng, ours.node(k)), _dense(eng, ref.node(k)))
        for dims in [(0,), (len(shape) - 1,)]:
            np.testing.assert_array_equal(_dense(eng, rwops.downsample_mean(src, dims)),
                                          _dense(eng, cc.ops.downsample_mean(src, dims)))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,chunk,levels", [((64, 64, 64), (32, 32, 32), 2),   # resident path
                                                ((40, 36, 28), (16, 16, 16), 2),   # streaming, ragged
                                                ((96, 80), (32, 32), 3)])
def test_engine_hierarchy_equals_device_path(shape, chunk, levels):
    import torch

    from paper_2509_26213_b200 import device
    from paper_2509_26213_b200.config import RWConfig

    vol = synthetic.phantom(shape)
    sd = synthetic.seeds(shape, "S1")
    pyr = rwops.hierarchical_random_walker(cc.ops.source_from_array(vol, chunk),
                                           cc.ops.source_from_array(sd, chunk), levels=levels, tol=1e-7)
    labels = rwops.rw_labels(pyr.node(0))
    with _engine() as eng:
        p_engine = _dense(eng, pyr.node(0))
        l_engine = _dense(eng, labels)
    res = device.hierarchical_random_walker(torch.from_numpy(vol).cuda(), torch.from_numpy(sd).cuda(), chunk,
                                            levels, RWConfig(tol=1e-7))
    torch.cuda.synchronize()
    # same kernels, same brick decomposition, same bound values -> same bytes
    np.testing.assert_array_equal(p_engine, res.prob.cpu().numpy())
    np.testing.assert_array_equal(l_engine, res.labels.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("per_task", [1, 64])
def test_engine_batching_is_transparent(per_task):
    """Engine-level batching: the random-walker operator solves each batch of
    chunk requests as one brick-list solve over the batch's union window; any batch size gives
    the bytes of the device path."""
    import torch
    from chunkcast.engine import Engine, EngineConfig
    from chunkcast.store import StoreConfig

    from paper_2509_26213_b200 import _native, device
    from paper_2509_26213_b200.config import RWConfig

    shape, chunk = (96, 64, 64), (32, 32, 32)
    vol = synthetic.phantom(shape)
    sd = synthetic.seeds(shape, "S1")
    pyr = rwops.hierarchical_random_walker(cc.ops.source_from_array(vol, chunk), cc.ops.source_from_array(sd, chunk),
                                           levels=2, tol=1e-7)
    lib = _native.lib()
    with Engine(EngineConfig(stores=StoreConfig(ram_capacity=1 << 28), worker_pool_size=2,
                             max_requests_per_task=per_task)) as eng:
        n0 = lib.rwb_kernel_launches()
        p_engine = _dense(eng, pyr.node(0))
        launches = lib.rwb_kernel_launches() - n0
    res = device.hierarchical_random_walker(torch.from_numpy(vol).cuda(), torch.from_numpy(sd).cuda(), chunk, 2,
                                            RWConfig(tol=1e-7))
    np.testing.assert_array_equal(p_engine, res.prob.cpu().numpy())
    assert launches > 0


@pytest.mark.gpu
def test_engine_weights_match_oracle():
    from oracle import rw as orw

    vol = synthetic.phantom((20, 18, 12))
    node = rwops.rw_weights(cc.ops.source_from_array(vol, (8, 8, 8)), 100.0, 1e-6)
    with _engine() as eng:
        w = _dense(eng, node)
    ref = orw.edge_weights(vol, 100.0, 1e-6)
    for k in range(3):
        np.testing.assert_allclose(w[..., k], ref[k], rtol=5e-6, atol=1e-12)


@pytest.mark.gpu
def test_engine_pull_is_lazy():
    shape, chunk = (128, 64, 64), (32, 32, 32)
    vol = cc.ops.source_from_array(synthetic.phantom(shape), chunk)
    sd = cc.ops.source_from_array(synthetic.seeds(shape), chunk)
    pyr = rwops.hierarchical_random_walker(vol, sd, levels=2)
    with _engine() as eng:
        eng.resolve_one(pyr.node(0), (0, 0, 0))
        # only the parent chunks under the dilated footprint of brick (0,0,0)
        assert eng.stats.requested_positions(pyr.node(0), pyr.node(1)) == {(0, 0, 0)}
        assert eng.stats.computed(pyr.node(0)) == 1


def test_rasterize_seeds_balls_and_conflicts():
    src = cc.ops.source_from_array(np.zeros((20, 24, 18), np.float32), (8, 8, 8))
    node = rwops.rasterize_seeds([(5, 6, 7), (15, 20, 3)], [(5, 8, 7), (0, 0, 0)], src, radius=2.0)
    assert node.md.element_type == cc.model.U8 and node.md.size == src.md.size
    with cc.engine.Engine(cc.engine.EngineConfig(stores=cc.store.StoreConfig(ram_capacity=1 << 26))) as eng:
        got = _dense(eng, node)
    g = np.stack(np.meshgrid(*[np.arange(n) for n in src.md.size], indexing="ij"), -1).astype(float)

    def ball(p):
        return ((g - np.array(p)) ** 2).sum(-1) <= 4.0

    fg = ball((5, 6, 7)) | ball((15, 20, 3))
    bg = ball((5, 8, 7)) | ball((0, 0, 0))
    want = np.where(fg & ~bg, 1, np.where(bg & ~fg, 2, 0)).astype(np.uint8)
    np.testing.assert_array_equal(got, want)
    assert (want == 0)[fg & bg].all() and (fg & bg).any()
    same = rwops.rasterize_seeds([(5, 6, 7), (15, 20, 3)], [(5, 8, 7), (0, 0, 0)], src, radius=2.0)
    assert same.op_id == node.op_id
    assert rwops.rasterize_seeds([(5, 6, 7)], [], src).op_id != node.op_id
    with pytest.raises(cc.ops.OperatorError):
        rwops.rasterize_seeds([(1, 2)], [], src)
