"""Drop-in operators for the reference compute graph (`chunkcast`, operator mode).

Factories in the idiom of `chunkcast.ops` (`pkg/src/chunkcast/ops.py`): pure
functions returning reference `OperatorNode`s (`graph.py:18-51`) whose
per-chunk `kernel(h, input_arrays, out)` runs the sm_100a kernels of librwb.
A reference `Engine` resolves them unchanged: it calls `dependencies(h)`,
pins the input chunks in RAM and runs the kernel on a worker thread
(`engine.py:999-1076`); the kernel stages the chunk neighbourhood to the
GPU, calls the C ABI and writes the result (including zero padding, as
`ops.py:517-520` requires) into `out`.  The random-walker operator instead carries a
`task_body` (engine-level batching): the engine hands it a batch of up to
`max_requests_per_task` chunk requests, and the batch becomes ONE brick-list solve over the
union window of its footprints (one upload, one launch sequence) instead of one solve per chunk.

    import chunkcast
    from paper_2509_26213_b200 import ops as rw

    vol = chunkcast.ops.source_from_array(volume, (32, 32, 32))
    seeds = chunkcast.ops.source_from_array(seed_labels, (32, 32, 32))
    prob = rw.hierarchical_random_walker(vol, seeds, levels=4)   # LodPyramid of p_fg
    labels = rw.rw_labels(prob.node(0))
    engine.resolve(labels)

Names and argument meaning follow the reference (`build_lod`,
`downsample`-style footprints, `OperatorError` for invalid graphs); results
are bit-identical to the device-batched path (`device.py`), which is the
throughput path this operator mode wraps chunk by chunk.

The reference package itself is needed (it owns `OperatorNode`/`Engine`):
it is imported from the environment or from `baseline/_ref`.
"""

from __future__ import annotations

import math
import os
import sys

import threading

import numpy as np

from .config import RWConfig

_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _chunkcast():
    try:
        import chunkcast  # noqa: F401
    except ImportError:
        ref = os.path.join(_ROOT, "baseline", "_ref")
        if os.path.isdir(os.path.join(ref, "chunkcast")) and ref not in sys.path:
            sys.path.append(ref)
        import chunkcast  # noqa: F401
    import chunkcast.graph
    import chunkcast.model
    import chunkcast.ops

    return chunkcast


def _error(msg):
    return _chunkcast().ops.OperatorError(msg)


# ---------------------------------------------------------------------------
# host-side chunk assembly (dtype preserving) and device staging


def _overlapping(md, begin, end):
    """Chunk positions of `md` intersecting the in-level region [begin, end)."""
    lo = [max(0, int(b)) // c for b, c in zip(begin, md.chunk_size)]
    hi = [-(-min(int(e), s) // c) for e, s, c in zip(end, md.size, md.chunk_size)]
    return [tuple(int(a + o) for a, o in zip(lo, off))
            for off in np.ndindex(*[max(h - l, 0) for l, h in zip(lo, hi)])]


def _gather(md, chunks: dict, begin, end) -> np.ndarray:
    """Copy the logical elements of [begin, end) out of padded chunk payloads."""
    shape = [e - b for b, e in zip(begin, end)]
    lanes = md.element_type.lanes
    out = np.empty(shape + ([lanes] if lanes > 1 else []), dtype=md.element_type.np_dtype)
    for h, payload in chunks.items():
        cb, ce = md.chunk_logical_region(h)
        lo = [max(a, c) for a, c in zip(begin, cb)]
        hi = [min(a, c) for a, c in zip(end, ce)]
        if any(x >= y for x, y in zip(lo, hi)):
            continue
        src = tuple(slice(a - c, b - c) for a, b, c in zip(lo, hi, cb))
        dst = tuple(slice(a - o, b - o) for a, b, o in zip(lo, hi, begin))
        out[dst] = payload[src]
    return out


def _write_out(out: np.ndarray, region_shape, values: np.ndarray):
    out[...] = 0
    out[tuple(slice(0, n) for n in region_shape)] = values


def _device():
    import torch

    from . import _native

    _native.lib()  # loud failure without the library / an sm_100 device
    return torch, torch.device("cuda", torch.cuda.current_device())


def _to_dev(a: np.ndarray):
    torch, dev = _device()
    a = np.ascontiguousarray(a)
    if not a.flags.writeable:  # engine-pinned input payloads are read-only views
        a = a.copy()
    return torch.from_numpy(a).to(dev)


def _from_dev(t) -> np.ndarray:
    import torch

    torch.cuda.current_stream().synchronize()
    return t.cpu().numpy()


def _dilated(md, h, r=1):
    begin, end = md.chunk_logical_region(h)
    return ([max(b - r, 0) for b in begin], [min(e + r, s) for e, s in zip(end, md.size)], begin, end)


# Device sections of the batched random-walker tasks run one at a time per process: the engine's
# worker threads still gather and scatter chunk payloads concurrently on the host, and the GPU
# work is one stream anyway, so interleaving them only adds allocator churn.
_DEVICE_LOCK = threading.Lock()


def _batched_body(ctx, inputs, dependencies, solve_batch):
    """Engine task body computing a whole batch of chunk requests in one call.

    The reference engine hands an operator's queued requests to one task in batches of up to
    `max_requests_per_task` (engine.py:790-816); its generic body then runs the operator's
    kernel once per chunk (`_generic_compute_body`, engine.py:999-1076).  This body keeps the
    generic body's input protocol (one deduplicated ChunkRequest per input, input states
    noted), but runs `solve_batch(positions, arrays)` — one device solve for the batch — as a
    single worker job, then stores every chunk's payload.
    """
    from chunkcast.engine import RAM, ChunkRequest, ChunkState, WorkerJob

    positions = [tuple(int(x) for x in p) for p in ctx.positions]
    per_input = [[] for _ in inputs]
    seen = [set() for _ in inputs]
    for pos in positions:
        for i, plist in enumerate(dependencies(pos)):
            for q in plist:
                q = tuple(q)
                if q not in seen[i]:
                    seen[i].add(q)
                    per_input[i].append(q)
    wanted = ChunkState.PREVIEW if ctx.wanted_state == ChunkState.PREVIEW else ChunkState.FINAL
    asked = [i for i, plist in enumerate(per_input) if plist]
    handle_lists = yield [ChunkRequest(inputs[i], per_input[i], RAM, min_state=wanted) for i in asked]
    arrays = [{} for _ in inputs]
    for i, handles in zip(asked, handle_lists):
        for q, h in zip(per_input[i], handles):
            arrays[i][q] = h.array
            ctx.note_input_state(h.state)
    results = yield WorkerJob(solve_batch, positions, arrays)
    for pos in positions:
        yield from ctx.store_chunk(pos, results[pos], ChunkState.FINAL)


def _check_f32(node, what):
    cc = _chunkcast()
    if node.md.element_type != cc.model.F32:
        raise _error(f"{what} must have scalar f32 elements, got {node.md.element_type}")


def _check_u8(node, what):
    cc = _chunkcast()
    if node.md.element_type != cc.model.U8:
        raise _error(f"{what} must have scalar u8 elements, got {node.md.element_type}")


# ---------------------------------------------------------------------------
# LOD pyramid


def lod_down(input_node):
    """Next coarser LOD level, fused conv([.25,.5,.25]^d, clamp) + 2x mean.

    Bit-identical to ``downsample_mean(separable_conv(node, [SMOOTHING_KERNEL]*d))``
    (`ops.py:714-727`), in one node and one GPU pass.
    """
    cc = _chunkcast()
    _check_f32(input_node, "lod_down input")
    md_in = input_node.md
    size = tuple(-(-s // 2) for s in md_in.size)
    md = cc.model.TensorMetaData(size, md_in.chunk_size, md_in.element_type)
    emb = None
    if input_node.embedding is not None:
        emb = cc.model.EmbeddingData(tuple(sp * 2 for sp in input_node.embedding.spacing))

    def src_window(h):
        # coarse [b, e) reads fine 2b-1 .. 2e (conv radius 1); start on an even
        # fine index so coarse j <-> fine 2j stays aligned in the window
        begin, end = md.chunk_logical_region(h)
        lo = [max(2 * b - 2, 0) for b in begin]
        hi = [min(2 * e + 2, s) for e, s in zip(end, md_in.size)]
        return lo, hi, begin, end

    def dependencies(h):
        lo, hi, _, _ = src_window(h)
        return [_overlapping(md_in, lo, hi)]

    def kernel(h, input_arrays, out):
        from . import device

        lo, hi, begin, end = src_window(h)
        block = _gather(md_in, dict(zip(dependencies(h)[0], input_arrays[0])), lo, hi)
        coarse = _from_dev(device.lod_down(_to_dev(block)))
        off = [b - l // 2 for b, l in zip(begin, lo)]
        sel = tuple(slice(o, o + e - b) for o, b, e in zip(off, begin, end))
        _write_out(out, [e - b for b, e in zip(begin, end)], coarse[sel])

    return cc.graph.OperatorNode(
        name="rwb.lod_down", params={"kernel": [0.25, 0.5, 0.25], "border": "clamp", "factor": 2},
        inputs=(input_node,), md=md, embedding=emb, dependencies=dependencies, kernel=kernel)


def downsample_mean(input_node, dims=None):
    """`chunkcast.ops.downsample_mean` on the GPU (`ops.py:611-676`): factor-2 mean over `dims`
    (default all), ceil sizes, a trailing odd element passing through, spacing x2 on the halved
    dimensions; float64 pairwise means rounded to f32, bit-identical to the reference."""
    cc = _chunkcast()
    _check_f32(input_node, "downsample_mean input")
    md_in = input_node.md
    d = md_in.num_dims
    sel = tuple(range(d)) if dims is None else tuple(sorted(dims))
    if any(not 0 <= k < d for k in sel):
        raise _error(f"downsample_mean dims {dims} outside a {d}-d tensor")
    size = tuple(-(-s // 2) if i in sel else s for i, s in enumerate(md_in.size))
    md = cc.model.TensorMetaData(size, md_in.chunk_size, md_in.element_type)
    emb = None
    if input_node.embedding is not None:
        emb = cc.model.EmbeddingData(tuple(sp * 2 if i in sel else sp
                                           for i, sp in enumerate(input_node.embedding.spacing)))

    def src_window(h):
        begin, end = md.chunk_logical_region(h)
        lo = [2 * b if i in sel else b for i, b in enumerate(begin)]
        hi = [min(2 * e, md_in.size[i]) if i in sel else e for i, e in enumerate(end)]
        return lo, hi, begin, end

    def dependencies(h):
        lo, hi, _, _ = src_window(h)
        return [_overlapping(md_in, lo, hi)]

    def kernel(h, input_arrays, out):
        from . import device

        lo, hi, begin, end = src_window(h)
        block = _gather(md_in, dict(zip(dependencies(h)[0], input_arrays[0])), lo, hi)
        coarse = _from_dev(device.downsample_mean(_to_dev(block), sel))
        _write_out(out, [e - b for b, e in zip(begin, end)], coarse)

    return cc.graph.OperatorNode(
        name="rwb.downsample_mean", params={"dims": [int(i) for i in sel]},
        inputs=(input_node,), md=md, embedding=emb, dependencies=dependencies, kernel=kernel)


def build_lod(input_node, embedding=None, smooth: bool = True, levels: int | None = None):
    """`chunkcast.ops.build_lod` with the fused GPU level step (`ops.py:714-727`).

    Same stop rule (halve until every dim fits one chunk) and the same level
    values: smooth=True chains the fused conv+mean `lod_down`, smooth=False the
    plain 2x mean (`downsample_mean`); `levels` optionally truncates the chain.
    """
    cc = _chunkcast()
    d = input_node.md.num_dims
    emb = embedding if embedding is not None else input_node.embedding
    if emb is None:
        emb = cc.model.EmbeddingData((1.0,) * d)
    elif not isinstance(emb, cc.model.EmbeddingData):
        emb = cc.model.EmbeddingData(tuple(emb))
    out = [(input_node, emb)]
    node = input_node
    while any(s > c for s, c in zip(node.md.size, node.md.chunk_size)):
        if levels is not None and len(out) >= levels:
            break
        node = lod_down(node) if smooth else downsample_mean(node)
        emb = cc.model.EmbeddingData(tuple(sp * 2 for sp in emb.spacing))
        out.append((node, emb))
    if levels is not None and len(out) < levels:
        raise _error(f"levels={levels} but the pyramid of {input_node.md.size} has only {len(out)} levels")
    return cc.ops.LodPyramid(tuple(out))


# ---------------------------------------------------------------------------
# random-walker operators


def rw_weights(volume_node, beta: float = 100.0, min_weight: float = 1e-6):
    """Forward edge weights max(exp(-beta dI^2), min_weight), F32 x ndim lanes (0 = no edge)."""
    cc = _chunkcast()
    _check_f32(volume_node, "rw_weights input")
    d = volume_node.md.num_dims
    if not 1 <= d <= 3:
        raise _error("rw_weights supports 1-3 dimensions")
    if not (beta >= 0 and min_weight >= 0):
        raise _error("beta and min_weight must be >= 0")
    md = cc.model.TensorMetaData(volume_node.md.size, volume_node.md.chunk_size, cc.model.Scalar.F32.vec(d)) \
        if d > 1 else cc.model.TensorMetaData(volume_node.md.size, volume_node.md.chunk_size, cc.model.F32)
    md_in = volume_node.md

    def window(h):
        begin, end = md.chunk_logical_region(h)
        return list(begin), [min(e + 1, s) for e, s in zip(end, md_in.size)], begin, end

    def dependencies(h):
        lo, hi, _, _ = window(h)
        return [_overlapping(md_in, lo, hi)]

    def kernel(h, input_arrays, out):
        from . import device

        lo, hi, begin, end = window(h)
        block = _gather(md_in, dict(zip(dependencies(h)[0], input_arrays[0])), lo, hi)
        w = _from_dev(device.edge_weights(_to_dev(block), beta, min_weight))
        # edges leaving the window but not the level were computed inside it;
        # the window's last slab only exists to give the region's forward edges
        sel = tuple(slice(0, e - b) for b, e in zip(begin, end))
        vals = w[sel] if d > 1 else w[sel][..., 0]
        _write_out(out, [e - b for b, e in zip(begin, end)], vals)

    return cc.graph.OperatorNode(
        name="rwb.weights", params={"beta": float(beta), "min_weight": float(min_weight)},
        inputs=(volume_node,), md=md, embedding=volume_node.embedding, dependencies=dependencies, kernel=kernel)


def project_seeds(seeds_node):
    """Seed labels of the next coarser level (fg/bg if only fg/bg children, conflicts -> 0)."""
    cc = _chunkcast()
    _check_u8(seeds_node, "project_seeds input")
    md_in = seeds_node.md
    md = cc.model.TensorMetaData(tuple(-(-s // 2) for s in md_in.size), md_in.chunk_size, cc.model.U8)

    def window(h):
        begin, end = md.chunk_logical_region(h)
        return [2 * b for b in begin], [min(2 * e, s) for e, s in zip(end, md_in.size)], begin, end

    def dependencies(h):
        lo, hi, _, _ = window(h)
        return [_overlapping(md_in, lo, hi)]

    def kernel(h, input_arrays, out):
        from . import device

        lo, hi, begin, end = window(h)
        block = _gather(md_in, dict(zip(dependencies(h)[0], input_arrays[0])), lo, hi)
        _write_out(out, [e - b for b, e in zip(begin, end)], _from_dev(device.project_seeds(_to_dev(block))))

    emb = None
    if seeds_node.embedding is not None:
        emb = cc.model.EmbeddingData(tuple(sp * 2 for sp in seeds_node.embedding.spacing))
    return cc.graph.OperatorNode(name="rwb.project_seeds", params={"rule": "conflict->unseeded"},
                                 inputs=(seeds_node,), md=md, embedding=emb, dependencies=dependencies,
                                 kernel=kernel)


def _parent_window(lo, hi, parent_size):
    """Parent index window the prolongation taps of fine [lo, hi) read (per dim)."""
    out_lo, out_hi = [], []
    for a, b, m in zip(lo, hi, parent_size):
        ja = a // 2
        first = ja if a % 2 else max(ja - 1, 0)
        jb = (b - 1) // 2
        last = min(jb + 1, m - 1) if (b - 1) % 2 else jb
        out_lo.append(first)
        out_hi.append(last + 1)
    return out_lo, out_hi


def random_walker(volume_node, seeds_node, parent=None, *, beta: float = 100.0, min_weight: float = 1e-6,
                  tol: float = 1e-6, max_iter: int = 10_000):
    """Random-walker foreground probability of one pyramid level (F32).

    Without `parent` the level is one Dirichlet problem (the coarsest level;
    every chunk request solves the whole level).  With `parent` (the F32
    probability node of the next coarser level) every chunk is an
    independent brick problem bounded and initialised by the upsampled
    parent solution.
    """
    cc = _chunkcast()
    _check_f32(volume_node, "random_walker volume")
    _check_u8(seeds_node, "random_walker seeds")
    md_in = volume_node.md
    if seeds_node.md.size != md_in.size or seeds_node.md.chunk_size != md_in.chunk_size:
        raise _error("volume and seeds must share size and chunking")
    if md_in.num_dims not in (2, 3):
        raise _error("the random walker supports 2-D and 3-D tensors")
    if parent is not None:
        _check_f32(parent, "random_walker parent")
        if parent.md.size != tuple(-(-s // 2) for s in md_in.size):
            raise _error("parent must be the next coarser level (size ceil(size/2))")
    cfg = RWConfig(beta=float(beta), min_weight=float(min_weight), tol=float(tol), max_iter=int(max_iter))
    md = cc.model.TensorMetaData(md_in.size, md_in.chunk_size, cc.model.F32)
    inputs = (volume_node, seeds_node) + ((parent,) if parent is not None else ())

    def dependencies(h):
        if parent is None:
            every = list(md_in.chunk_positions())
            return [every, every]
        lo, hi, _, _ = _dilated(md, h)
        plo, phi = _parent_window(lo, hi, parent.md.size)
        vol = _overlapping(md_in, lo, hi)
        return [vol, vol, _overlapping(parent.md, plo, phi)]

    payload_shape = md.element_type.payload_shape(md.chunk_size)
    # whole-level solution of a coarsest-level node, computed by the first batch that needs it
    # (the operator is a pure function of its inputs, so later batches reuse it)
    whole, whole_lock = [], threading.Lock()

    def solve_batch(positions, arrays):
        """Probability payloads of a batch of chunks from one device solve (engine-level
        batching): the union window of the chunks' footprints is gathered
        and uploaded once, and every chunk is one brick of a single brick-list solve."""
        from . import _native, device

        nd = md.num_dims
        out = {}
        if parent is None:  # the coarsest level: one whole-level solve serves every batch
            with whole_lock:
                if not whole:
                    lo, hi = [0] * nd, list(md.size)
                    vol = _gather(md_in, arrays[0], lo, hi)
                    sd = _gather(seeds_node.md, arrays[1], lo, hi)
                    with _DEVICE_LOCK:
                        prob, _ = device.solve_level(_to_dev(vol), _to_dev(sd), tuple(md.size), None, cfg)
                        whole.append(_from_dev(prob))
                p = whole[0]
            for h in positions:
                begin, end = md.chunk_logical_region(h)
                o = np.empty(payload_shape, np.float32)
                _write_out(o, [e - b for b, e in zip(begin, end)], p[tuple(slice(b, e) for b, e in zip(begin, end))])
                out[h] = o
            return out
        boxes = [_dilated(md, h) for h in positions]
        lo = [min(b[0][d] for b in boxes) for d in range(nd)]
        hi = [max(b[1][d] for b in boxes) for d in range(nd)]
        vol = _gather(md_in, arrays[0], lo, hi)
        sd = _gather(seeds_node.md, arrays[1], lo, hi)
        plo, phi = _parent_window(lo, hi, parent.md.size)
        par = _gather(parent.md, arrays[2], plo, phi)
        with _DEVICE_LOCK:
            p = _solve_window(vol, sd, par, lo, hi, plo, phi, positions)
        for h, (_, _, begin, end) in zip(positions, boxes):
            o = np.empty(payload_shape, np.float32)
            _write_out(o, [e - b for b, e in zip(begin, end)],
                       p[tuple(slice(b - a, e - a) for a, b, e in zip(lo, begin, end))])
            out[h] = o
        return out

    def _solve_window(vol, sd, par, lo, hi, plo, phi, positions):
        from . import _native, device

        nd = md.num_dims
        torch, dev = _device()
        win = [b - a for a, b in zip(lo, hi)]
        bound = torch.empty(win, dtype=torch.float32, device=dev)
        par_d = _to_dev(par)
        a64 = _native.int64_array
        _native.check(_native.lib().rwb_upsample_window_f32(
            nd, a64(parent.md.size), a64(plo), a64([b - a for a, b in zip(plo, phi)]),
            device._ptr(par_d), a64(md.size), a64(lo), a64(win), device._ptr(bound), device._stream_handle()))
        # the window's brick grid is the chunk grid shifted by the window origin
        brick = tuple(md.chunk_size)
        origin = tuple(-(a % c) for a, c in zip(lo, brick))
        grid = device.brick_grid(win, brick, origin)
        index = []
        for h in positions:
            i = 0
            for hd, a, c, gdim in zip(h, lo, brick, grid):
                i = i * gdim + (hd - a // c)
            index.append(i)
        blist = torch.tensor(index, dtype=torch.int32, device=dev)
        prob, _ = device.solve_level(_to_dev(vol), _to_dev(sd), brick, bound, cfg, brick_list=blist, origin=origin)
        return _from_dev(prob)

    def task_body(ctx):
        return _batched_body(ctx, inputs, dependencies, solve_batch)

    return cc.graph.OperatorNode(
        name="rwb.random_walker", params=dict(cfg.params(), hierarchical=parent is not None),
        inputs=inputs, md=md, embedding=volume_node.embedding, dependencies=dependencies, task_body=task_body)


def hierarchical_random_walker(volume_node, seeds_node, levels: int | None = None, *, beta: float = 100.0,
                               min_weight: float = 1e-6, tol: float = 1e-6, max_iter: int = 10_000,
                               embedding=None):
    """Pyramid of random-walker probabilities, level 0 finest (`LodPyramid`).

    Coarsest level solved whole, every finer level brick by brick from the
    upsampled level above — pulled lazily: resolving chunk h of level 0 only
    computes the parent chunks its footprint needs.
    """
    cc = _chunkcast()
    vol_pyr = build_lod(volume_node, embedding=embedding, levels=levels)
    n = vol_pyr.num_levels
    seeds = [seeds_node]
    for _ in range(n - 1):
        seeds.append(project_seeds(seeds[-1]))
    kw = dict(beta=beta, min_weight=min_weight, tol=tol, max_iter=max_iter)
    probs = [None] * n
    probs[n - 1] = random_walker(vol_pyr.node(n - 1), seeds[n - 1], None, **kw)
    for k in range(n - 2, -1, -1):
        probs[k] = random_walker(vol_pyr.node(k), seeds[k], probs[k + 1], **kw)
    return cc.ops.LodPyramid(tuple((probs[k], vol_pyr.embedding(k)) for k in range(n)))


def rasterize_seeds(fg_points, bg_points, md, radius: float = 0.0, embedding=None):
    """U8 seed labels {0, 1, 2} as a source node: voxel g is foreground (1)
    when ||g - p|| <= radius for a point p of `fg_points`, background (2) for `bg_points`, and
    unseeded (0) when it is in both or neither (the conflict rule of the seed projection).
    `md`: a reference `TensorMetaData` or a node whose metadata (size, chunking) the labels share.
    Points are voxel coordinates (d floats).  Identity is content-addressed like
    `source_from_array` (`ops.py:282-325`): equal point sets give equal operator ids.  Host-side
    rasterisation of a handful of balls per chunk; any U8 label node serves as seeds just as well."""
    cc = _chunkcast()
    if hasattr(md, "md"):
        md = md.md
    d = md.num_dims
    md = cc.model.TensorMetaData(tuple(md.size), tuple(md.chunk_size), cc.model.U8)
    pts = []
    for plist, what in ((fg_points, "fg_points"), (bg_points, "bg_points")):
        a = np.asarray(plist, dtype=np.float64) if len(plist) else np.zeros((0, d))
        if a.ndim != 2 or a.shape[1] != d:
            raise _error(f"{what} must hold {d}-d coordinates")
        pts.append(a)
    r = float(radius)
    if r < 0:
        raise _error("radius must be non-negative")

    def kernel(h, input_arrays, out):
        begin, end = md.chunk_logical_region(h)
        grids = np.meshgrid(*[np.arange(b, e, dtype=np.float64) for b, e in zip(begin, end)], indexing="ij")
        hit = []
        for a in pts:
            m = np.zeros(grids[0].shape, bool)
            for p in a:
                if all(pk + r >= b and pk - r <= e - 1 for pk, b, e in zip(p, begin, end)):
                    m |= sum((g - pk) ** 2 for g, pk in zip(grids, p)) <= r * r
            hit.append(m)
        lab = np.where(hit[0] & ~hit[1], 1, np.where(hit[1] & ~hit[0], 2, 0)).astype(np.uint8)
        _write_out(out, [e - b for b, e in zip(begin, end)], lab)

    return cc.graph.OperatorNode(
        name="rwb.rasterize_seeds",
        params={"fg": [[float(x) for x in p] for p in pts[0]], "bg": [[float(x) for x in p] for p in pts[1]],
                "radius": r, "size": [int(s) for s in md.size], "chunk": [int(c) for c in md.chunk_size]},
        inputs=(), md=md, embedding=embedding, dependencies=lambda h: [], kernel=kernel)


def rw_labels(prob_node):
    """Segmentation labels: 1 where p > 0.5, else 0 (U8)."""
    cc = _chunkcast()
    _check_f32(prob_node, "rw_labels input")
    md = cc.model.TensorMetaData(prob_node.md.size, prob_node.md.chunk_size, cc.model.U8)

    def dependencies(h):
        return [[tuple(h)]]

    def kernel(h, input_arrays, out):
        from . import device

        out[...] = _from_dev(device.labels(_to_dev(np.ascontiguousarray(input_arrays[0][0]))))

    return cc.graph.OperatorNode(name="rwb.labels", params={"threshold": 0.5}, inputs=(prob_node,), md=md,
                                 embedding=prob_node.embedding, dependencies=dependencies, kernel=kernel)


def level_voxels(pyramid) -> int:
    return math.prod(pyramid.node(0).md.size)
