"""Pan/zoom views (viewer half): `render.slice_view` / `image_view` on device
pyramids against the reference's own `chunkcast.render.slice_view` / `image_view` resolved by its
Engine — byte-identical frames."""

import numpy as np
import pytest

from conftest import reference_package

from paper_2509_26213_b200 import ops as rwops
from paper_2509_26213_b200.render import zoom_level

cc = reference_package()  # fails (does not skip) when the reference is missing


def test_zoom_level_rule():
    assert zoom_level(1.0, 4) == 0 and zoom_level(0.5, 4) == 1 and zoom_level(0.3, 4) == 1
    assert zoom_level(0.25, 4) == 2 and zoom_level(4.0, 4) == 0 and zoom_level(1e-6, 4) == 3
    with pytest.raises(ValueError):
        zoom_level(0.0, 3)


def _frame(eng, node):
    out = np.zeros(node.md.element_type.payload_shape(node.md.size), node.md.element_type.np_dtype)
    pos = list(node.md.chunk_positions())
    for p, a in zip(pos, eng.resolve(node, pos)):
        b, e = node.md.chunk_logical_region(p)
        out[tuple(slice(x, y) for x, y in zip(b, e))] = a[tuple(slice(0, y - x) for x, y in zip(b, e))]
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("dim,index,pan,zoom", [(0, 17, (0.0, 0.0), 1.0), (1, 40, (-3.5, 7.25), 0.6),
                                                (2, 63, (10.0, -20.0), 2.5), (0, 5, (1.0, 2.0), 0.2)])
def test_slice_view_matches_reference(dim, index, pan, zoom):
    import torch
    from chunkcast import render as rr
    from chunkcast.engine import Engine, EngineConfig
    from chunkcast.model import TensorMetaData, F32
    from chunkcast.store import StoreConfig

    from paper_2509_26213_b200 import device, render, synthetic

    vol = torch.from_numpy(synthetic.phantom((48, 64, 64))).cuda()
    levels = device.lod_chain(vol, (16, 16, 16))
    frame_size, tile = (50, 70), (16, 32)
    ours = render.slice_view(levels, dim, index, pan, zoom, frame_size).cpu().numpy()
    pyr = cc.ops.LodPyramid(tuple((cc.ops.source_from_array(lv.cpu().numpy(), (16, 16, 16)),
                                   cc.model.EmbeddingData((2.0 ** k,) * 3)) for k, lv in enumerate(levels)))
    node = rr.slice_view(pyr, dim, index, pan, zoom, TensorMetaData(frame_size, tile, F32))
    with Engine(EngineConfig(stores=StoreConfig(ram_capacity=1 << 27))) as eng:
        ref = _frame(eng, node)
    np.testing.assert_array_equal(ours, ref)


@pytest.mark.gpu
@pytest.mark.parametrize("pan,zoom", [((0.0, 0.0), 1.0), ((-5.0, 3.0), 0.45), ((20.0, 11.0), 3.0)])
def test_image_view_matches_reference(pan, zoom):
    import torch
    from chunkcast import render as rr
    from chunkcast.engine import Engine, EngineConfig
    from chunkcast.model import TensorMetaData, U8
    from chunkcast.store import StoreConfig

    from paper_2509_26213_b200 import render, synthetic

    labels = torch.from_numpy((synthetic.phantom((96, 80)) > 0.5).astype(np.uint8)).cuda()
    levels = [labels, labels[::2, ::2].contiguous(), labels[::4, ::4].contiguous()]
    frame_size, tile = (40, 64), (16, 16)
    ours = render.image_view(levels, pan, zoom, frame_size).cpu().numpy()
    pyr = cc.ops.LodPyramid(tuple((cc.ops.source_from_array(lv.cpu().numpy(), (32, 32)),
                                   cc.model.EmbeddingData((2.0 ** k,) * 2)) for k, lv in enumerate(levels)))
    node = rr.image_view(pyr, pan, zoom, TensorMetaData(frame_size, tile, U8))
    with Engine(EngineConfig(stores=StoreConfig(ram_capacity=1 << 27))) as eng:
        ref = _frame(eng, node)
    np.testing.assert_array_equal(ours, ref)


# -- volume raycaster (render.py:101-631) ----------------------------------------------


def test_camera_and_projection_match_reference():
    from chunkcast import render as rr
    from chunkcast.model import EmbeddingData, TensorMetaData, F32

    from paper_2509_26213_b200 import render

    md = TensorMetaData((40, 36, 28), (16, 16, 16), F32)
    spacing = (1.0, 0.5, 2.0)
    cam = rr.camera_for_volume(md, EmbeddingData(spacing), fov_deg=40.0)
    ours = render.fit_camera(md.size, spacing, fov_deg=40.0)
    assert np.allclose(ours["eye"], cam.eye) and np.allclose(ours["look_at"], cam.look_at)
    assert ours["near"] == cam.near and ours["far"] == cam.far
    np.testing.assert_array_equal(render.view_projection(ours, 1.5), rr.view_projection(cam, 1.5))


@pytest.mark.gpu
@pytest.mark.parametrize("compositing,u8,bias,sdf,tf", [("dvr", True, 0.0, 0.5, (0.0, 1.0)),
                                                        ("dvr", False, 0.0, 0.5, (0.05, 0.6)),
                                                        ("mop", True, 0.0, 1.0, (0.0, 1.0)),
                                                        ("dvr", True, 1.0, 0.7, (0.1, 0.9))])
def test_raycast_matches_reference(compositing, u8, bias, sdf, tf):
    """The GPU raycaster against the reference's render_frame resolved by its Engine (final frame,
    float64 march in both, the same operations in the same order): byte-identical frames."""
    import torch
    from chunkcast import render as rr
    from chunkcast.engine import Engine, EngineConfig
    from chunkcast.model import RGBA_F32, RGBA_U8
    from chunkcast.store import StoreConfig

    from paper_2509_26213_b200 import device, render, synthetic

    shape, chunk = (40, 48, 36), (16, 16, 16)
    vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
    levels = device.lod_chain(vol, chunk)
    frame_size, tile = (56, 72), (16, 24)
    camera = render.fit_camera(shape, (1.0, 1.0, 1.0), fov_deg=50.0)
    ours = render.raycast_frame(levels, (1.0, 1.0, 1.0), frame_size, camera, compositing=compositing,
                                sample_distance_factor=sdf, lod_bias=bias, tf=tf, u8=u8, tile=tile)
    ours = ours.cpu().numpy()
    pyr = cc.ops.build_lod(cc.ops.source_from_array(vol.cpu().numpy(), chunk))
    cfg = rr.RaycasterConfig(compositing=compositing, sample_distance_factor=sdf, lod_bias=bias)
    cam = rr.CameraState(**camera)
    with Engine(EngineConfig(stores=StoreConfig(ram_capacity=1 << 28))) as eng:
        ref = rr.render_frame(eng, pyr, cam, cfg, rr.grey_ramp_tf(*tf), frame_size, tile,
                              element_type=RGBA_U8 if u8 else RGBA_F32)
    assert ours.shape == ref.shape and ours.dtype == ref.dtype
    assert (ref[..., 3] > 0).mean() > 0.2  # the volume covers a good part of the frame
    np.testing.assert_array_equal(ours, ref)
