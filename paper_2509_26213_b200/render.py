"""Pan/zoom views of probability (or intensity) pyramids on the GPU — SURVEY.md §8(f)4, the
viewer half of the reference's `render.py`.

`slice_view` and `image_view` restate `render.py:634-741`: the pyramid level is the one where a
frame pixel covers at least one source element (`_zoom_level`: floor(-log2 zoom), clipped), and
every frame pixel p samples source element floor((p + 0.5) * scale + offset) with
scale = 1 / (zoom * 2^level) and offset = pan / 2^level (`_resample_nn`), 0 outside the source.
Here the levels are device tensors and one `rwb_resample_nn` launch fills the whole frame (the
reference resolves it tile by tile through its engine); the frames are byte-identical to the
reference's (tests/test_render.py).  The raycaster (`render.py:203-631`) is not part of this
module.
"""

from __future__ import annotations

import ctypes
import math

import torch

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
