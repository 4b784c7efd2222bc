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


def segment_many(inputs, brick=(32, 32, 32), levels=None, cfg: RWConfig = RWConfig(), *, outputs=None,
                 workspace: device.Workspace | None = None):
    """Segment a sequence of host volumes with the transfers overlapped.

    `inputs`: list of (volume, seeds) host tensors of one shape (pinned for
    asynchronous copies); `outputs`: optional list of (prob, labels) pinned
    host tensors, reused cyclically when shorter than `inputs`.  Volume k+1 is
    uploaded on its own stream while volume k is segmented, and the results
    of volume k are downloaded on a third stream while volume k+1 is
    segmented (device inputs double-buffered), so in steady state a volume
    costs max(upload, compute, download) instead of their sum.  Returns the
    list of (prob, labels) host tensors, complete when the call returns.
    """
    n = len(inputs)
    if n == 0:
        return []
    dev = torch.device("cuda", torch.cuda.current_device())
    comp = torch.cuda.current_stream(dev)
    up = torch.cuda.Stream(dev)
    down = torch.cuda.Stream(dev)
    up.wait_stream(comp)
    down.wait_stream(comp)
    shape = tuple(inputs[0][0].shape)
    vol_d = [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(min(n, 2))]
    sd_d = [torch.empty(shape, dtype=torch.uint8, device=dev) for _ in range(min(n, 2))]
    if outputs is None:
        outputs = [(torch.empty(shape, dtype=torch.float32, pin_memory=True),
                    torch.empty(shape, dtype=torch.uint8, pin_memory=True)) for _ in range(min(n, 2))]
    computed = []

    def upload(i):
        b = i % 2
        with torch.cuda.stream(up):
            if i >= 2:
                up.wait_event(computed[i - 2])  # buffer b is free once volume i-2 is segmented
            v, s = inputs[i]
            vol_d[b].copy_(_as_host_tensor(v, np.float32), non_blocking=True)
            sd_d[b].copy_(_as_host_tensor(s, np.uint8), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(up)
        return ev

    uploaded = [upload(0)]
    results = []
    for i in range(n):
        if i + 1 < n:
            uploaded.append(upload(i + 1))
        comp.wait_event(uploaded[i])
        res = device.hierarchical_random_walker(vol_d[i % 2], sd_d[i % 2], brick, levels, cfg,
                                                workspace=workspace)
        ev = torch.cuda.Event()
        ev.record(comp)
        computed.append(ev)
        out_p, out_l = outputs[i % len(outputs)]
        with torch.cuda.stream(down):
            down.wait_event(ev)
            out_p.copy_(res.prob, non_blocking=True)
            out_l.copy_(res.labels, non_blocking=True)
            res.prob.record_stream(down)
            res.labels.record_stream(down)
        results.append((out_p, out_l))
    comp.wait_stream(down)
    comp.wait_stream(up)
    comp.synchronize()
    return results
