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
            workspace: device.Workspace | None = None, pyramid_store=None, pyramid_key=None, roi=None):
    """Hierarchical random-walker segmentation.

    volume: float32 intensities (numpy or torch, host or CUDA); seeds: uint8
    labels (0 none, 1 foreground, 2 background) of the same shape.  Returns
    (probabilities f32, labels u8) on the device the inputs came from: host
    inputs get host outputs (written into `out_prob` / `out_labels` when
    given, e.g. pinned buffers).  `pyramid_store` (a store.DeviceStore) with `pyramid_key`
    keeps the volume's LOD pyramid in HBM under a budget, so segmenting the same volume again
    (new seeds or parameters) skips rebuilding it.  `roi` = (lo, hi) level-0 voxel box: only the
    bricks that region needs are solved on every level, and (prob, labels) of the box are returned
    (identical to the same box of a full segmentation).
    """
    vol = _as_host_tensor(volume, np.float32)
    sd = _as_host_tensor(seeds, np.uint8)
    if roi is not None:
        dev = vol.device if vol.is_cuda else torch.device("cuda", torch.cuda.current_device())
        res = device.hierarchical_random_walker(vol.to(dev, non_blocking=True), sd.to(dev, non_blocking=True), brick,
                                                levels, cfg, workspace=workspace, pyramid_store=pyramid_store,
                                                pyramid_key=pyramid_key, roi=roi)
        box = tuple(slice(max(0, int(a)), int(b)) for a, b in zip(roi[0], roi[1]))
        p, lab = res.prob[box], res.labels[box]
        if vol.is_cuda:
            return p, lab
        return p.cpu(), lab.cpu()
    if vol.is_cuda:
        res = device.hierarchical_random_walker(vol, sd, brick, levels, cfg, workspace=workspace,
                                                pyramid_store=pyramid_store, pyramid_key=pyramid_key)
        return res.prob, res.labels
    if out_prob is None:
        out_prob = torch.empty(tuple(vol.shape), dtype=torch.float32, pin_memory=True)
    if out_labels is None:
        out_labels = torch.empty(tuple(vol.shape), dtype=torch.uint8, pin_memory=True)
    # one volume through the overlapped pipeline: level-0 slabs download while the rest solves
    return segment_many([(vol, sd)], brick, levels, cfg, outputs=[(out_prob, out_labels)], workspace=workspace,
                        pyramid_store=pyramid_store, pyramid_keys=[pyramid_key])[0]


def segment_many(inputs, brick=(32, 32, 32), levels=None, cfg: RWConfig = RWConfig(), *, outputs=None,
                 workspace: device.Workspace | None = None, level0_chunks: int | None = None, pyramid_store=None,
                 pyramid_keys=None, cyclic_outputs: bool = False, store=None, input_ids=None):
    """Segment a sequence of host volumes with the transfers overlapped.

    `inputs`: list of (volume, seeds) host tensors of one shape (pinned for
    asynchronous copies); `outputs`: optional list of (prob, labels) pinned
    host tensors, one pair per input (default: allocated here).  A shorter
    list is an error unless `cyclic_outputs=True`, which reuses the pairs
    cyclically (later volumes overwrite earlier results: a throughput probe
    that does not keep them).  Volume k+1 is
    uploaded on its own stream while volume k is segmented, and the results
    of volume k are downloaded on a third stream while volume k+1 is
    segmented (device inputs double-buffered), so in steady state a volume
    costs max(upload, compute, download) instead of their sum; level 0 is
    solved in `level0_chunks` slabs whose rows download while the next slab
    solves, so even the last volume's download mostly overlaps its compute.  Returns the
    list of (prob, labels) host tensors, complete when the call returns.

    `store` (a store.DeviceStore): the device copies of the inputs live in the store's HBM arena
    under its budget instead of a private double buffer — one entry per input (volume bytes then
    seed bytes, key `input_ids[i]`), reserved and uploaded one volume ahead, pinned while
    segmented, then retired on the compute stream, so the LRU / epoch GC recycles them once their
    work has run.  Inputs already resident (same id) are not uploaded again.
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
    nvox = 1
    for d in shape:
        nvox *= int(d)
    if store is None:
        vol_d = [torch.empty(shape, dtype=torch.float32, device=dev) for _ in range(min(n, 2))]
        sd_d = [torch.empty(shape, dtype=torch.uint8, device=dev) for _ in range(min(n, 2))]
    else:
        vol_d, sd_d = [None] * n, [None] * n
        held = [None] * n  # pinned store entries
        if input_ids is None:
            input_ids = [("segment_many", id(v), id(sd), i) for i, (v, sd) in enumerate(inputs)]
    if outputs is None:
        outputs = [(torch.empty(shape, dtype=torch.float32, pin_memory=True),
                    torch.empty(shape, dtype=torch.uint8, pin_memory=True)) for _ in range(n)]
    elif len(outputs) < n and not cyclic_outputs:
        raise ValueError(f"{len(outputs)} output pairs for {n} inputs (pass cyclic_outputs=True to reuse them)")
    elif len(outputs) == 0:
        raise ValueError("outputs is empty")
    computed = []

    def upload(i):
        if store is not None:
            return upload_to_store(i)
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

    def upload_to_store(i):
        from .store import ChunkState

        got = store.get(input_ids[i], torch.uint8, (5 * nvox,))
        if got is not None:  # resident: no transfer
            e, payload = got
            ev = None
        else:
            e = store.reserve(input_ids[i], 5 * nvox)  # may evict retired inputs (their work has run)
            payload = e.payload
            with torch.cuda.stream(up):
                v, s = inputs[i]
                payload[: 4 * nvox].view(torch.float32).view(shape).copy_(_as_host_tensor(v, np.float32),
                                                                         non_blocking=True)
                payload[4 * nvox:].view(shape).copy_(_as_host_tensor(s, np.uint8), non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
            e.state = ChunkState.FINAL
        held[i] = e
        vol_d[i] = payload[: 4 * nvox].view(torch.float32).view(shape)
        sd_d[i] = payload[4 * nvox:].view(shape)
        return ev

    uploaded = [upload(0)]
    results = []
    for i in range(n):
        if i + 1 < n:
            uploaded.append(upload(i + 1))
        if uploaded[i] is not None:
            comp.wait_event(uploaded[i])
        out_p, out_l = outputs[i % len(outputs)]
        slot = i if store is not None else i % 2

        def download(r0, r1, prob, labels, out_p=out_p, out_l=out_l):
            # level-0 rows [r0, r1) are final at this point of the compute stream:
            # download them while the remaining slabs solve
            ev_c = torch.cuda.Event()
            ev_c.record(torch.cuda.current_stream())  # the stream that produced the rows
            with torch.cuda.stream(down):
                down.wait_event(ev_c)
                out_p[r0:r1].copy_(prob[r0:r1], non_blocking=True)
                out_l[r0:r1].copy_(labels[r0:r1], non_blocking=True)
                prob.record_stream(down)
                labels.record_stream(down)

        device.hierarchical_random_walker(vol_d[slot], sd_d[slot], brick, levels, cfg, workspace=workspace,
                                          level0_chunks=level0_chunks, on_level0_chunk=download,
                                          pyramid_store=pyramid_store,
                                          pyramid_key=pyramid_keys[i] if pyramid_keys is not None else None)
        ev = torch.cuda.Event()
        ev.record(comp)
        computed.append(ev)
        results.append((out_p, out_l))
        if store is not None:  # collectable once this volume's work has run
            store.retire(held[i], comp)
            held[i] = vol_d[i] = sd_d[i] = None
    comp.wait_stream(down)
    comp.wait_stream(up)
    comp.synchronize()
    return results


def segment_series(volume, seeds, brick=(32, 32, 32), levels=None, cfg: RWConfig = RWConfig(), *,
                   outputs=None, workspace: device.Workspace | None = None, store=None, series_id=None):
    """Per-timestep hierarchical random walker of a 4-D (T, Z, Y, X) host series.

    The reference's 4-D → 3-D `slice_node` view (`ops.py:555-586`), one
    timestep at a time: every timestep is a host view streamed through
    `segment_many` (upload of t+1 and download of t-1 overlapped with t), so
    only two timesteps are ever resident on the device — the series may be far
    larger than HBM.  Returns (prob, labels) host tensors of shape (T, ...);
    `outputs` = (prob, labels) pinned 4-D buffers to write into.  With `store`
    (a store.DeviceStore whose budget may be far below the series) the timesteps
    stream through the store's arena as entries (series_id, t): evicted LRU-first
    once segmented, still resident — and not uploaded again — on a later call
    while the budget holds them.
    """
    vol = _as_host_tensor(volume, np.float32)
    sd = _as_host_tensor(seeds, np.uint8)
    if vol.dim() < 2 or vol.shape != sd.shape:
        raise ValueError("volume and seeds must be (T, ...) series of the same shape")
    if outputs is None:
        outputs = (torch.empty(tuple(vol.shape), dtype=torch.float32, pin_memory=True),
                   torch.empty(tuple(vol.shape), dtype=torch.uint8, pin_memory=True))
    prob, labels = outputs
    n = vol.shape[0]
    sid = series_id if series_id is not None else ("series", vol.data_ptr(), sd.data_ptr(), tuple(vol.shape))
    segment_many([(vol[t], sd[t]) for t in range(n)], brick, levels, cfg,
                 outputs=[(prob[t], labels[t]) for t in range(n)], workspace=workspace, store=store,
                 input_ids=[(sid, t) for t in range(n)] if store is not None else None)
    return prob, labels
