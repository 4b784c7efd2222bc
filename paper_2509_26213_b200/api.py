"""Public entry points of the hot path.

`segment` is the call a user makes: host (or device) volume and seeds in,
probabilities and labels out.  With host inputs it stages them through
pinned memory onto the current CUDA device, runs the hierarchical random
walker (`device.hierarchical_random_walker`) and copies the results back;
this is the end-to-end path `bench.py` times for its `e2e` number.
"""

from __future__ import annotations

import numpy as np
import torch

from . import device
from .config import RWConfig


def _as_host_tensor(a, dtype):
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype))
    if isinstance(a, torch.Tensor):
        return a
    raise TypeError("expected a numpy array or torch tensor")


def segment(volume, seeds, brick=(32, 32, 32), levels=None, cfg: RWConfig = RWConfig(), *,
            out_prob: torch.Tensor | None = None, out_labels: torch.Tensor | None = None,
            workspace: device.Workspace | None = None):
    """Hierarchical random-walker segmentation.

    volume: float32 intensities (numpy or torch, host or CUDA); seeds: uint8
    labels (0 none, 1 foreground, 2 background) of the same shape.  Returns
    (probabilities f32, labels u8) on the device the inputs came from: host
    inputs get host outputs (written into `out_prob` / `out_labels` when
    given, e.g. pinned buffers).
    """
    vol = _as_host_tensor(volume, np.float32)
    sd = _as_host_tensor(seeds, np.uint8)
    on_host = not vol.is_cuda
    dev = torch.device("cuda", torch.cuda.current_device())
    if on_host:
        vol_d = vol.to(dev, non_blocking=vol.is_pinned())
        sd_d = sd.to(dev, non_blocking=sd.is_pinned())
    else:
        vol_d, sd_d = vol, sd
    res = device.hierarchical_random_walker(vol_d, sd_d, brick, levels, cfg, workspace=workspace)
    if not on_host:
        return res.prob, res.labels
    if out_prob is None:
        out_prob = torch.empty(res.prob.shape, dtype=torch.float32, pin_memory=True)
    if out_labels is None:
        out_labels = torch.empty(res.labels.shape, dtype=torch.uint8, pin_memory=True)
    out_prob.copy_(res.prob, non_blocking=out_prob.is_pinned())
    out_labels.copy_(res.labels, non_blocking=out_labels.is_pinned())
    torch.cuda.current_stream().synchronize()
    return out_prob, out_labels
