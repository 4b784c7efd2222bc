"""Pan/zoom views of probability (or intensity) pyramids on the GPU — SURVEY.md §8(f)4, the
viewer half of the reference's `render.py`.

`slice_view` and `image_view` restate `render.py:634-741`: the pyramid level is the one where a
frame pixel covers at least one source element (`_zoom_level`: floor(-log2 zoom), clipped), and
every frame pixel p samples source element floor((p + 0.5) * scale + offset) with
scale = 1 / (zoom * 2^level) and offset = pan / 2^level (`_resample_nn`), 0 outside the source.
Here the levels are device tensors and one `rwb_resample_nn` launch fills the whole frame (the
reference resolves it tile by tile through its engine); the frames are byte-identical to the
reference's (tests/test_render.py).

`raycast_frame` is the volume raycaster (`render.py:101-631`): the per-pixel ray records (the
reference's camera, view-projection, `_pixel_rays`, `_slab_clip` and its entry-exit node's float32
storage, computed here with the same float64 numpy expressions) go to `rwb_raycast`, which marches
every pixel on the GPU (csrc/rwb_render.cu) over the device-resident pyramid.
"""

from __future__ import annotations

import ctypes
import math

import torch

import numpy as np

from . import _native, device


def zoom_level(zoom: float, num_levels: int) -> int:
    """Pyramid level for `zoom` screen pixels per level-0 element (`render.py:634-637`)."""
    if not zoom > 0:
        raise ValueError("zoom must be positive")
    return int(min(max(math.floor(-math.log2(zoom)), 0), num_levels - 1))


def _resample(src: torch.Tensor, slice_dim: int, slice_index: int, frame_size, scale, offset) -> torch.Tensor:
    if not src.is_cuda:
        raise ValueError("the pyramid levels must be CUDA tensors")
    src = src.contiguous()
    frame = torch.empty(tuple(int(f) for f in frame_size), dtype=src.dtype, device=src.device)
    dbl2 = ctypes.c_double * 2
    _native.check(_native.lib().rwb_resample_nn(
        src.dim(), _native.int64_array(src.shape), int(slice_dim), int(slice_index), src.element_size(),
        device._ptr(src), _native.int64_array(frame.shape), dbl2(*[float(s) for s in scale]),
        dbl2(*[float(o) for o in offset]), device._ptr(frame), device._stream_handle()))
    return frame


def slice_view(levels, dim: int, index: int, pan, zoom: float, frame_size) -> torch.Tensor:
    """Axis-aligned slice of a 3-D pyramid (list of device tensors, level 0 finest) under pan/zoom
    (`render.py:703-728`): `pan` is the level-0 element coordinate at frame pixel (0, 0)."""
    base = levels[0]
    if base.dim() != 3:
        raise ValueError("slice view needs a 3-D source")
    if not 0 <= dim < 3:
        raise ValueError(f"slice dim {dim} out of range")
    if not 0 <= index < base.shape[dim]:
        raise ValueError(f"slice index {index} out of range for size {base.shape[dim]}")
    level = zoom_level(zoom, len(levels))
    node = levels[level]
    idx = min(index >> level, node.shape[dim] - 1)
    factor = float(1 << level)
    scale = (1.0 / (zoom * factor),) * 2
    offset = tuple(float(p) / factor for p in pan)
    return _resample(node, dim, idx, frame_size, scale, offset)


def image_view(levels, pan, zoom: float, frame_size) -> torch.Tensor:
    """Pan/zoom view of a 2-D pyramid (`render.py:731-741`)."""
    if levels[0].dim() != 2:
        raise ValueError("image view needs a 2-D pyramid")
    level = zoom_level(zoom, len(levels))
    factor = float(1 << level)
    scale = (1.0 / (zoom * factor),) * 2
    offset = tuple(float(p) / factor for p in pan)
    return _resample(levels[level], -1, 0, frame_size, scale, offset)


# ---------------------------------------------------------------------------
# volume raycasting (render.py:70-631)

_EPS_UP = 1e-12


def fit_camera(volume_size, spacing, fov_deg: float = 45.0) -> dict:
    """The reference's auto camera (`camera_for_volume`, `render.py:101-119`): eye on the box
    diagonal at the distance where the bounding sphere spans the vertical fov."""
    phys = np.asarray([n * s for n, s in zip(volume_size, spacing)], np.float64)
    center = phys / 2.0
    radius = float(np.linalg.norm(phys)) / 2.0
    dist = radius / math.tan(math.radians(fov_deg) / 2.0)
    eye = center + dist * (np.ones(3) / math.sqrt(3.0))
    return dict(eye=tuple(eye), look_at=tuple(center), up=(0.0, 0.0, 1.0), fov_deg=float(fov_deg),
                near=max(1e-3 * radius, dist - 2.0 * radius), far=dist + 2.0 * radius)


def view_projection(camera: dict, aspect: float) -> np.ndarray:
    """Right-handed look-at times perspective, NDC z in [-1, 1] (`render.py:122-142`)."""
    eye = np.asarray(camera["eye"], np.float64)
    fwd = np.asarray(camera["look_at"], np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(camera.get("up", (0.0, 0.0, 1.0)), np.float64))
    right /= np.linalg.norm(right)
    up = np.cross(right, fwd)
    view = np.eye(4)
    view[0, :3], view[1, :3], view[2, :3] = right, up, -fwd
    view[:3, 3] = -view[:3, :3] @ eye
    fy = 1.0 / math.tan(math.radians(camera.get("fov_deg", 45.0)) / 2.0)
    n, f = camera.get("near", 0.01), camera.get("far", 100.0)
    proj = np.zeros((4, 4))
    proj[0, 0], proj[1, 1] = fy / aspect, fy
    proj[2, 2], proj[2, 3], proj[3, 2] = (f + n) / (n - f), 2.0 * f * n / (n - f), -1.0
    return proj @ view


def _to_world(inv_vp, ndc):
    h = np.concatenate([ndc, np.ones(ndc.shape[:-1] + (1,))], axis=-1) @ inv_vp.T
    return h[..., :3] / h[..., 3:4]


def _tile_records(inv_vp, frame_size, r0, r1, c0, c1, extent):
    hgt, wdt = int(frame_size[0]), int(frame_size[1])
    rows, cols = np.meshgrid(np.arange(r0, r1, dtype=np.float64), np.arange(c0, c1, dtype=np.float64), indexing="ij")
    ndc = np.stack([(cols + 0.5) / wdt * 2.0 - 1.0, 1.0 - (rows + 0.5) / hgt * 2.0], axis=-1)
    near = _to_world(inv_vp, np.concatenate([ndc, np.full(ndc.shape[:-1] + (1,), -1.0)], -1))
    far = _to_world(inv_vp, np.concatenate([ndc, np.full(ndc.shape[:-1] + (1,), 1.0)], -1))
    seg = far - near
    length = np.linalg.norm(seg, axis=-1)
    direction = seg / length[..., None]
    probe = np.array([[0.0, 0.0], [2.0 / wdt, 0.0]])
    pn = _to_world(inv_vp, np.concatenate([probe, np.full((2, 1), -1.0)], -1))
    pf = _to_world(inv_vp, np.concatenate([probe, np.full((2, 1), 1.0)], -1))
    pitch_near = float(np.linalg.norm(pn[1] - pn[0]))
    pitch_far = float(np.linalg.norm(pf[1] - pf[0]))
    fp0 = np.full_like(length, pitch_near)
    fps = (pitch_far - pitch_near) / length
    ext = np.asarray(extent, np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / direction
        t0 = (0.0 - near) * inv
        t1 = (ext - near) * inv
    lo, hi = np.minimum(t0, t1), np.maximum(t0, t1)
    par = direction == 0.0
    inside = (near >= 0.0) & (near <= ext)
    lo = np.where(par, np.where(inside, -np.inf, np.inf), lo)
    hi = np.where(par, np.where(inside, np.inf, -np.inf), hi)
    t_in = np.maximum(lo.max(axis=-1), 0.0)
    t_out = np.minimum(hi.min(axis=-1), length)
    miss = t_in > t_out
    t_in = np.where(miss, np.inf, t_in)
    t_out = np.where(miss, -np.inf, t_out)
    eep = np.stack([t_in, t_out, fp0, fps], axis=-1).astype(np.float32).astype(np.float64)
    return np.concatenate([near, direction, eep], axis=-1)


def ray_records(matrix, frame_size, extent, tile=(64, 64)) -> np.ndarray:
    """Per pixel (row-major): origin (3), unit direction (3), then the entry-exit record
    (t_entry, t_exit, fp0, fps) rounded through float32 as the reference's entry-exit node stores
    it (`render.py:162-249`); misses get t_entry = +inf, t_exit = -inf.  Computed tile by tile
    (`tile` = the frame chunking), the array shapes the reference evaluates the same numpy
    expressions on, so even the BLAS products round identically."""
    inv_vp = np.linalg.inv(np.asarray(matrix, np.float64))
    hgt, wdt = int(frame_size[0]), int(frame_size[1])
    out = np.empty((hgt, wdt, 10))
    for r0 in range(0, hgt, tile[0]):
        for c0 in range(0, wdt, tile[1]):
            r1, c1 = min(r0 + tile[0], hgt), min(c0 + tile[1], wdt)
            out[r0:r1, c0:c1] = _tile_records(inv_vp, (hgt, wdt), r0, r1, c0, c1, extent)
    return out.reshape(hgt * wdt, 10)


def raycast_frame(levels, spacing, frame_size, camera=None, *, compositing: str = "dvr",
                  sample_distance_factor: float = 0.5, lod_bias: float = 0.0, tf=(0.0, 1.0),
                  u8: bool = True, tile=(64, 64)) -> torch.Tensor:
    """Raycast a frame of a 3-D pyramid (device tensors, level 0 finest; level k spacing =
    `spacing` x 2^k as `build_lod` assigns): the final frame of the reference's `render_frame`
    with `RaycasterConfig(compositing, sample_distance_factor, lod_bias)` and `grey_ramp_tf(*tf)`.
    `camera`: None (the fitted camera), a dict of CameraState fields, or a 4x4 view-projection.
    Returns (H, W, 4) premultiplied RGBA, u8 or float32, on the levels' device."""
    if compositing not in ("dvr", "mop"):
        raise ValueError("compositing must be 'dvr' or 'mop'")
    base = levels[0]
    if base.dim() != 3 or not base.is_cuda:
        raise ValueError("the raycaster needs a 3-D CUDA pyramid")
    hgt, wdt = int(frame_size[0]), int(frame_size[1])
    if camera is None:
        camera = fit_camera(base.shape, spacing)
    matrix = view_projection(camera, wdt / hgt) if isinstance(camera, dict) else np.asarray(camera, np.float64)
    extent = [n * s for n, s in zip(base.shape, spacing)]
    rays = torch.from_numpy(ray_records(matrix, (hgt, wdt), extent, tile)).to(base.device)
    lv = [t.contiguous() for t in levels]
    n = len(lv)
    ptrs = (ctypes.c_void_p * n)(*[ctypes.c_void_p(t.data_ptr()) for t in lv])
    sizes = _native.int64_array([int(x) for t in lv for x in t.shape])
    sp = (ctypes.c_double * (3 * n))(*[float(s) * (1 << k) for k in range(n) for s in spacing])
    out = torch.empty((hgt, wdt, 4), dtype=torch.uint8 if u8 else torch.float32, device=base.device)
    _native.check(_native.lib().rwb_raycast(
        n, ptrs, sizes, sp, hgt * wdt, device._ptr(rays), 1 if compositing == "mop" else 0,
        float(sample_distance_factor), float(lod_bias), float(tf[0]), float(tf[1]), 1 if u8 else 0,
        device._ptr(out), device._stream_handle()))
    return out
