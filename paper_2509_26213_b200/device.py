"""Device-resident hot path: torch tensors in HBM -> librwb kernels.

PyTorch only provides device memory and the current CUDA stream; every
arithmetic step runs in the hand-written sm_100a kernels of librwb.so
(`csrc/`), called through the C ABI of `include/rwb.h`.

Level layout in HBM: one dense row-major tensor per pyramid level (f32
intensity, u8 seeds, f32 probabilities), exactly the logical tensors of the
reference's `TensorMetaData` (model.py:98-177); bricks are windows of the
chunk grid.  The solver's brick-local workspace is a caller-owned uint8
tensor (`Workspace`), reused across levels.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import torch

from . import _native
from .config import RWConfig


def _stream_handle():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr() if t is not None else 0)


def _check_tensor(t: torch.Tensor, dtype, name: str, ndim=None):
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the random-walker path has no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if ndim is not None and t.dim() not in ndim:
        raise ValueError(f"{name} must have {ndim} dims, got {t.dim()}")


def coarse_shape(shape):
    return tuple(-(-int(s) // 2) for s in shape)


# ---------------------------------------------------------------------------
# per-voxel operators


def lod_down(level: torch.Tensor) -> torch.Tensor:
    """Next coarser LOD level (bit-identical to the reference's conv+downsample)."""
    _check_tensor(level, torch.float32, "level", (1, 2, 3))
    lib = _native.lib()
    out = torch.empty(coarse_shape(level.shape), dtype=torch.float32, device=level.device)
    _native.check(lib.rwb_lod_down_f32(level.dim(), _native.int64_array(level.shape), _ptr(level), _ptr(out),
                                       _stream_handle()))
    return out


def downsample_mean(level: torch.Tensor, dims=None) -> torch.Tensor:
    """Factor-2 mean downsampling alone (the reference's build_lod(smooth=False) step,
    `downsample_mean`, ops.py:611-676; float64 pairwise means rounded to f32, bit-identical).
    `dims`: the dimensions to halve (default all), as `downsample_mean(input, dims)`."""
    _check_tensor(level, torch.float32, "level", (1, 2, 3))
    nd = level.dim()
    sel = tuple(range(nd)) if dims is None else tuple(sorted({int(d) for d in dims}))
    if any(d < 0 or d >= nd for d in sel):
        raise ValueError(f"dims {dims} outside a {nd}-d level")
    lib = _native.lib()
    shape = [-(-s // 2) if d in sel else s for d, s in enumerate(level.shape)]
    out = torch.empty(shape, dtype=torch.float32, device=level.device)
    mask = sum(1 << d for d in sel)
    _native.check(lib.rwb_downsample_mean_dims_f32(nd, _native.int64_array(level.shape), mask, _ptr(level),
                                                   _ptr(out), _stream_handle()))
    return out


def num_lod_levels(shape, chunk) -> int:
    """Level count of the reference's `build_lod` stop rule (ops.py:720)."""
    shape = [int(s) for s in shape]
    n = 1
    while any(s > c for s, c in zip(shape, chunk)):
        shape = [-(-s // 2) for s in shape]
        n += 1
    return n


def lod_chain(volume: torch.Tensor, chunk, levels: int | None = None) -> list:
    total = num_lod_levels(volume.shape, chunk)
    levels = total if levels is None else int(levels)
    if not 1 <= levels <= total:
        raise ValueError(f"levels={levels} outside 1..{total} for size {tuple(volume.shape)}, chunk {tuple(chunk)}")
    out = [volume]
    for _ in range(levels - 1):
        out.append(lod_down(out[-1]))
    return out


def _cached_lod_chain(volume, chunk, levels, store, key):
    """`lod_chain` with levels 1.. kept in a DeviceStore (store.py) under (key, k): segmenting the
    same volume again (new seeds, new parameters) reuses its pyramid from HBM while the store's
    budget lets it stay; evicted levels are recomputed and re-inserted."""
    total = num_lod_levels(volume.shape, chunk)
    n = total if levels is None else int(levels)
    if not 1 <= n <= total:
        raise ValueError(f"levels={n} outside 1..{total} for size {tuple(volume.shape)}, chunk {tuple(chunk)}")
    vols = [volume]
    held = []
    for k in range(1, n):
        shape = coarse_shape(vols[-1].shape)
        got = store.get((key, k), torch.float32, shape)
        if got is not None:
            held.append(got[0])
            vols.append(got[1])
            continue
        lv = lod_down(vols[-1])
        store.put((key, k), lv)
        vols.append(lv)
    for e in held:  # views stay valid: the stream orders any later reuse after this solve's reads
        store.unpin(e)
    return vols


def project_seeds(seeds: torch.Tensor) -> torch.Tensor:
    _check_tensor(seeds, torch.uint8, "seeds", (1, 2, 3))
    lib = _native.lib()
    out = torch.empty(coarse_shape(seeds.shape), dtype=torch.uint8, device=seeds.device)
    _native.check(lib.rwb_project_seeds_u8(seeds.dim(), _native.int64_array(seeds.shape), _ptr(seeds), _ptr(out),
                                           _stream_handle()))
    return out


def upsample(parent: torch.Tensor, fine_shape, out: torch.Tensor | None = None) -> torch.Tensor:
    _check_tensor(parent, torch.float32, "parent", (1, 2, 3))
    fine_shape = tuple(int(s) for s in fine_shape)
    if out is None:
        out = torch.empty(fine_shape, dtype=torch.float32, device=parent.device)
    _check_tensor(out, torch.float32, "out")
    if tuple(out.shape) != fine_shape:
        raise ValueError("out has the wrong shape")
    lib = _native.lib()
    _native.check(lib.rwb_upsample_f32(parent.dim(), _native.int64_array(parent.shape), _ptr(parent),
                                       _native.int64_array(fine_shape), _ptr(out), _stream_handle()))
    return out


def upsample_planes(parent: torch.Tensor, parent_z0: int, fine_shape, g0: int, g1: int, out: torch.Tensor,
                    out_z0: int = 0) -> torch.Tensor:
    """Fine planes [g0, g1) (dim 0, global indices) of a level of global shape `fine_shape`, from a
    parent window: `parent` holds the parent level's global planes [parent_z0, parent_z0 +
    parent.shape[0]) and must cover their prolongation taps (sharding.parent_planes).  `out`
    holds the fine global planes [out_z0, out_z0 + out.shape[0]).  Same values as `upsample`."""
    _check_tensor(parent, torch.float32, "parent", (2, 3))
    _check_tensor(out, torch.float32, "out")
    fine_shape = tuple(int(s) for s in fine_shape)
    if g1 <= g0:
        return out
    if g0 < out_z0 or g1 > out_z0 + out.shape[0] or tuple(out.shape[1:]) != fine_shape[1:]:
        raise ValueError("out does not hold the requested planes")
    nd = parent.dim()
    psize = coarse_shape(fine_shape)
    a64 = _native.int64_array
    view = out[g0 - out_z0:g1 - out_z0]
    _native.check(_native.lib().rwb_upsample_window_f32(
        nd, a64(psize), a64([parent_z0] + [0] * (nd - 1)), a64(parent.shape), _ptr(parent), a64(fine_shape),
        a64([g0] + [0] * (nd - 1)), a64([g1 - g0] + list(fine_shape[1:])), _ptr(view), _stream_handle()))
    return out


def upsample_window(parent: torch.Tensor, fine_shape, z0: int, z1: int, out: torch.Tensor) -> torch.Tensor:
    """Upsample only planes [z0, z1) (dim 0) of the fine level into `out` (full fine shape)."""
    _check_tensor(parent, torch.float32, "parent", (2, 3))
    _check_tensor(out, torch.float32, "out")
    fine_shape = tuple(int(s) for s in fine_shape)
    if tuple(out.shape) != fine_shape:
        raise ValueError("out has the wrong shape")
    if z1 <= z0:
        return out
    nd = parent.dim()
    fo = [z0] + [0] * (nd - 1)
    fw = [z1 - z0] + list(fine_shape[1:])
    view = out[z0:z1]
    lib = _native.lib()
    a64 = _native.int64_array
    _native.check(lib.rwb_upsample_window_f32(nd, a64(parent.shape), a64([0] * nd), a64(parent.shape), _ptr(parent),
                                              a64(fine_shape), a64(fo), a64(fw), _ptr(view), _stream_handle()))
    return out


def edge_weights(volume: torch.Tensor, beta: float = 100.0, min_weight: float = 1e-6) -> torch.Tensor:
    """Forward edge weights, lanes-last: shape volume.shape + (ndim,)."""
    _check_tensor(volume, torch.float32, "volume", (1, 2, 3))
    lib = _native.lib()
    out = torch.empty(tuple(volume.shape) + (volume.dim(),), dtype=torch.float32, device=volume.device)
    _native.check(lib.rwb_edge_weights_f32(volume.dim(), _native.int64_array(volume.shape), _ptr(volume),
                                           float(beta), float(min_weight), _ptr(out), _stream_handle()))
    return out


def labels(prob: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    _check_tensor(prob, torch.float32, "prob")
    if out is None:
        out = torch.empty(prob.shape, dtype=torch.uint8, device=prob.device)
    _check_tensor(out, torch.uint8, "out")
    lib = _native.lib()
    _native.check(lib.rwb_labels_u8(prob.numel(), _ptr(prob), _ptr(out), _stream_handle()))
    return out


# ---------------------------------------------------------------------------
# level solve


class Workspace:
    """Grow-only device scratch buffer for the brick solver."""

    def __init__(self, device=None):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.buffer = None

    def get(self, nbytes: int) -> torch.Tensor:
        if self.buffer is None or self.buffer.numel() < nbytes:
            self.buffer = None
            self.buffer = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        return self.buffer

    def release(self):
        self.buffer = None


def geometry(shape, brick, origin=None) -> _native.Geometry:
    nd = len(shape)
    if nd not in (2, 3):
        raise ValueError("the random walker supports 2-D and 3-D levels")
    if len(brick) != nd:
        raise ValueError("brick dimensionality mismatch")
    g = _native.Geometry()
    g.ndim = nd
    origin = origin or (0,) * nd
    for i in range(nd):
        g.size[i] = int(shape[i])
        g.brick[i] = int(brick[i])
        g.origin[i] = int(origin[i])
    return g


def brick_grid(shape, brick, origin=None):
    origin = origin or (0,) * len(shape)
    return tuple(-(-(int(s) - int(o)) // int(b)) for s, b, o in zip(shape, brick, origin))


def _flags(cfg: RWConfig) -> int:
    f = 0 if cfg.use_graph else _native.SOLVE_NO_GRAPH
    if not cfg.resident:
        f |= _native.SOLVE_STREAMING
    if not cfg.cooperative:
        f |= _native.SOLVE_NO_COOP
    if cfg.multigrid is False:
        f |= _native.SOLVE_NO_MG
    elif cfg.multigrid is True:
        f |= _native.SOLVE_MG
    if not cfg.coarse:
        f |= _native.SOLVE_NO_COARSE
    if not cfg.fused_setup:
        f |= _native.SOLVE_SETUP2
    if cfg.cluster == 4:  # 4-CTA clusters, weights in shared memory
        f |= _native.SOLVE_CLUSTER4
    elif cfg.cluster == 16:
        f |= _native.SOLVE_CLUSTER16
    elif cfg.cluster == 512:  # 8-CTA clusters, 512 threads per CTA
        f |= _native.SOLVE_SPLIT_Z
    elif cfg.cluster != 8:
        raise ValueError("cluster must be 4, 8, 16 or 512")
    return f


def workspace_bytes(shape, brick, n_bricks=-1, origin=None, cfg: RWConfig = RWConfig()) -> int:
    g = geometry(shape, brick, origin)
    return int(_native.load_library().rwb_solve_workspace_bytes(ctypes.byref(g), int(n_bricks), _flags(cfg)))


def solve_level(volume: torch.Tensor, seeds: torch.Tensor, brick, bound: torch.Tensor | None = None,
                cfg: RWConfig = RWConfig(), *, brick_list: torch.Tensor | None = None, out: torch.Tensor | None = None,
                labels_out: torch.Tensor | None = None, workspace: Workspace | None = None,
                origin=None, phase: str | None = None, stats_on_device: bool = False) -> tuple:
    """Random-walker solve of (the listed bricks of) one level.

    `bound` = upsampled parent probabilities (Dirichlet values outside each
    brick and initial guess); None only when `brick` covers the level.
    `out` may be `bound` itself (in-place).  Returns (prob, stats dict).
    `phase` ("setup" / "solve", brick-resident levels only) splits the call in two:
    "setup" builds the system in the workspace, a later "solve" with the same
    arguments and workspace solves it (stats only from "solve").
    `stats_on_device`: the stats are written by the device into pinned host memory
    without a host synchronisation; the returned `DeviceStats` resolves to the dict
    once the stream has passed the solve (`.resolve()`).
    """
    _check_tensor(volume, torch.float32, "volume", (2, 3))
    _check_tensor(seeds, torch.uint8, "seeds")
    if seeds.shape != volume.shape:
        raise ValueError("seeds and volume shapes differ")
    if bound is not None:
        _check_tensor(bound, torch.float32, "bound")
        if bound.shape != volume.shape:
            raise ValueError("bound and volume shapes differ")
    if out is None:
        out = torch.empty(volume.shape, dtype=torch.float32, device=volume.device)
    _check_tensor(out, torch.float32, "out")
    if labels_out is not None:
        _check_tensor(labels_out, torch.uint8, "labels_out")
    n_list = -1
    if brick_list is not None:
        _check_tensor(brick_list, torch.int32, "brick_list", (1,))
        n_list = brick_list.numel()
    g = geometry(volume.shape, brick, origin)
    if bound is None and any(n > 1 for n in brick_grid(volume.shape, brick, origin)):
        raise ValueError("a brick-wise solve needs `bound` (the upsampled parent level)")
    lib = _native.lib()
    nbytes = int(lib.rwb_solve_workspace_bytes(ctypes.byref(g), n_list, _flags(cfg)))
    if nbytes == 0:
        raise ValueError(f"invalid solver geometry: {_native.load_library().rwb_last_error().decode()}")
    workspace = workspace or Workspace(volume.device)
    ws = workspace.get(nbytes)
    p = _native.SolveParams()
    p.beta, p.min_weight, p.tol = float(cfg.beta), float(cfg.min_weight), float(cfg.tol)
    p.max_iter, p.check_every = int(cfg.max_iter), int(cfg.check_every)
    p.flags = _flags(cfg) | {None: 0, "setup": _native.SOLVE_SETUP_ONLY, "solve": _native.SOLVE_NO_SETUP}[phase]
    if stats_on_device and phase != "setup":
        p.flags |= _native.SOLVE_STATS_DEVICE
        dstats = DeviceStats()
        _native.check(lib.rwb_solve_level(
            ctypes.byref(g), _ptr(volume), _ptr(seeds), _ptr(bound), _ptr(brick_list), int(max(n_list, 0)),
            ctypes.byref(p), _ptr(out), _ptr(labels_out), _ptr(ws), ctypes.c_size_t(ws.numel()),
            ctypes.c_void_p(dstats.buffer.data_ptr()), _stream_handle()))
        return out, dstats
    stats = _native.SolveStats()
    _native.check(lib.rwb_solve_level(
        ctypes.byref(g), _ptr(volume), _ptr(seeds), _ptr(bound), _ptr(brick_list), int(max(n_list, 0)),
        ctypes.byref(p), _ptr(out), _ptr(labels_out), _ptr(ws), ctypes.c_size_t(ws.numel()),
        ctypes.byref(stats) if phase != "setup" else None, _stream_handle()))
    return out, (stats.as_dict() if phase != "setup" else None)


class DeviceStats:
    """Solver stats written by the device into pinned (device-mapped) host memory."""

    def __init__(self):
        self.buffer = torch.zeros(ctypes.sizeof(_native.SolveStats), dtype=torch.uint8, pin_memory=True)

    def resolve(self) -> dict:
        """The stats dict; the caller must have synchronised past the solve."""
        return _native.SolveStats.from_buffer_copy(self.buffer.numpy().tobytes()).as_dict()


def _resolve(st):
    return st.resolve() if isinstance(st, DeviceStats) else st


# ---------------------------------------------------------------------------
# hierarchical driver


def _merge_stats(parts):
    parts = [_resolve(s) for s in parts]
    out = dict(parts[0])
    for s in parts[1:]:
        for key in ("bricks", "converged", "not_converged", "zero_rhs", "iterations_sum", "unknowns",
                    "unknown_iterations"):
            out[key] += s[key]
        for key in ("iterations_max", "sweeps"):
            out[key] = max(out[key], s[key])
        out["cg_ms"] += s["cg_ms"]
    return out


def _solve_level_chunked(volume, seeds, brick, parent, cfg, labels_out, workspace, chunks, on_chunk, *,
                         z0: int = 0, fine_shape=None, parent_z0: int = 0, origin_z: int = 0, n_rows=None):
    """One level solved as `chunks` slabs of whole brick rows along dim 0, in order,
    all into the same output; `on_chunk(r0, r1, prob, labels)` is called after each slab's
    launches are queued (its rows [r0, r1) are final once the stream reaches
    that point), e.g. to queue the slab's download while the next one solves.  The
    bound (the upsampled `parent` level) is produced slab by slab (the slab's planes
    plus their one-plane halo), just before the slab's setup.

    Slab-local use (sharding.py): `volume` / `seeds` hold the global planes [z0, z0 + nz) of a
    level of global shape `fine_shape`, the solved brick rows start at local plane `origin_z`
    (the planes before it are Dirichlet halo) and `n_rows` of them are solved; `parent` holds the
    parent level's global planes from `parent_z0` on.  Defaults: the whole level."""
    fine_shape = tuple(volume.shape) if fine_shape is None else tuple(int(x) for x in fine_shape)
    # the ABI's brick grid origin lies in (-brick, 0]: a halo plane before the first solved row is
    # the tail of a brick row 0 that is not listed
    if not 0 <= origin_z < brick[0]:
        raise ValueError("origin_z must lie in [0, brick)")
    row0 = 1 if origin_z > 0 else 0
    origin = (origin_z - brick[0] if origin_z > 0 else 0,) + (0,) * (volume.dim() - 1)
    grid = brick_grid(volume.shape, brick, origin)
    per_row = math.prod(grid[1:])
    rows = grid[0] - row0 if n_rows is None else int(n_rows)
    chunks = max(1, min(chunks, rows))
    out = torch.empty(volume.shape, dtype=torch.float32, device=volume.device)
    parts = []
    bounds = [(rows * c // chunks, rows * (c + 1) // chunks) for c in range(chunks)]
    lists = [torch.arange((row0 + h0) * per_row, (row0 + h1) * per_row, dtype=torch.int32, device=volume.device)
             for h0, h1 in bounds]
    rows_of = [(origin_z + h0 * brick[0], min(origin_z + h1 * brick[0], volume.shape[0])) for h0, h1 in bounds]
    bound = torch.empty(volume.shape, dtype=torch.float32, device=volume.device)
    nz = volume.shape[0]

    def upsample_slab(c):  # the slab's planes + one-plane halo (identical bytes where slabs overlap)
        r0, r1 = rows_of[c]
        upsample_planes(parent, parent_z0, fine_shape, z0 + max(r0 - 1, 0), z0 + min(r1 + 1, nz), bound, z0)

    if not (cfg.resident and _resident_geometry(volume.shape, brick)):
        for c in range(chunks):
            upsample_slab(c)
            _, st = solve_level(volume, seeds, brick, bound, cfg, brick_list=lists[c], out=out, labels_out=labels_out,
                                workspace=workspace, origin=origin, stats_on_device=True)
            parts.append(st)
            if on_chunk is not None:
                on_chunk(*rows_of[c], out, labels_out)
        return out, parts
    # Brick-resident slabs, two-phase: slab c+1's system is built on a setup stream while slab
    # c solves on a high-priority stream (the engine's clusters leave SMs free for the setup
    # CTAs; priority hands SMs back to the engine first).  Two workspaces alternate.
    comp = torch.cuda.current_stream()
    solver = torch.cuda.Stream(priority=-1)
    setup = torch.cuda.Stream()
    solver.wait_stream(comp)
    setup.wait_stream(comp)
    spaces = [workspace, _twin(workspace)]
    done = [None, None]  # event after the last solve that used each workspace

    def build(c):
        with torch.cuda.stream(setup):
            upsample_slab(c)
            if done[c % 2] is not None:
                setup.wait_event(done[c % 2])
            solve_level(volume, seeds, brick, bound, cfg, brick_list=lists[c], out=out, labels_out=labels_out,
                        workspace=spaces[c % 2], origin=origin, phase="setup")
            ev = torch.cuda.Event()
            ev.record(setup)
        return ev

    built = build(0)
    for c in range(chunks):
        nxt = build(c + 1) if c + 1 < chunks else None
        with torch.cuda.stream(solver):
            solver.wait_event(built)
            _, st = solve_level(volume, seeds, brick, bound, cfg, brick_list=lists[c], out=out, labels_out=labels_out,
                                workspace=spaces[c % 2], origin=origin, phase="solve", stats_on_device=True)
            ev = torch.cuda.Event()
            ev.record(solver)
            done[c % 2] = ev
            parts.append(st)
            if on_chunk is not None:
                on_chunk(*rows_of[c], out, labels_out)
        built = nxt
    comp.wait_stream(solver)
    comp.wait_stream(setup)
    bound.record_stream(setup)
    out.record_stream(solver)
    if labels_out is not None:
        labels_out.record_stream(solver)
    return out, parts


def decided_bricks(bound: torch.Tensor, seeds: torch.Tensor, brick, eps: float) -> torch.Tensor:
    """The brick-skip rule (oracle/rw.py `decided_bricks`): True per brick (row-major) when the
    upsampled parent over the brick and its one-voxel halo is within `eps` of 0 or 1 everywhere
    (seeded voxels count as decided).  One max-pool over the level."""
    import torch.nn.functional as F

    amb = torch.minimum(bound, 1.0 - bound).masked_fill(seeds != 0, 0.0)
    nd = bound.dim()
    grid = brick_grid(bound.shape, brick)
    pool = F.max_pool3d if nd == 3 else F.max_pool2d
    m = pool(amb[None, None], kernel_size=tuple(b + 2 for b in brick), stride=tuple(brick), padding=1,
             ceil_mode=True)[0, 0]
    m = m[tuple(slice(0, g) for g in grid)]
    if tuple(m.shape) != tuple(grid):
        raise RuntimeError("brick-skip pooling does not match the brick grid")
    return (m < eps).reshape(-1)


def _solve_level_skipping(volume, seeds, brick, parent, cfg, want_labels, workspace):
    """One level under the brick-skip rule: the decided bricks keep the upsampled parent (seeds
    exact), the others are solved as a brick list."""
    bound = upsample(parent, volume.shape)
    skip = decided_bricks(bound, seeds, brick, cfg.skip_eps)
    out = torch.where(seeds == 1, torch.ones_like(bound), torch.where(seeds == 2, torch.zeros_like(bound), bound))
    todo = torch.nonzero(~skip).reshape(-1).to(torch.int32)
    nskip = int(skip.numel() - todo.numel())
    if todo.numel() == 0:
        return out, {"bricks": 0, "converged": 0, "not_converged": 0, "zero_rhs": 0, "iterations_max": 0,
                     "iterations_sum": 0, "unknowns": 0, "unknown_iterations": 0, "sweeps": 0, "cg_ms": 0.0,
                     "path": -1}, nskip
    _, st = solve_level(volume, seeds, brick, bound, cfg, brick_list=todo, out=out, workspace=workspace,
                        stats_on_device=True)
    return out, st, nskip


def _resident_geometry(shape, brick) -> bool:
    """Levels the brick-resident engines take (rwb_solve.cu use_resident)."""
    return (len(shape) == 3 and tuple(brick) == (32, 32, 32)) or (len(shape) == 2 and tuple(brick) == (64, 64))


def _twin(workspace):
    """A second workspace paired with `workspace` (kept on it, grown on demand)."""
    twin = getattr(workspace, "_twin", None)
    if twin is None:
        twin = Workspace(workspace.device)
        workspace._twin = twin
    return twin


@dataclass
class HRWResult:
    prob: torch.Tensor            # level-0 probabilities (f32)
    labels: torch.Tensor | None   # level-0 labels (u8, p > 0.5)
    levels: list                  # per-level probabilities, level 0 finest
    volumes: list                 # LOD pyramid used
    seeds: list                   # projected seeds per level
    stats: list = field(default_factory=list)  # per-level solver stats (level 0 first)


def roi_brick_boxes(shapes, brick, roi):
    """Lazy, region-limited hierarchy (the reference computes only the chunks a request needs,
    `engine.py:423-462`; Palace only the visible bricks, `PAPER.md:424`): per level k < L-1 the
    box [b0, b1) of brick coordinates to solve so that level 0 is exact inside `roi` = (lo, hi)
    (level-0 voxel coordinates).  Level k's listed bricks plus their one-voxel Dirichlet halo read
    the parent through the prolongation taps; the level-(k+1) bricks covering those taps are listed
    in turn.  The coarsest level is always whole (None)."""
    nd = len(shapes[0])
    lo = [max(0, int(a)) for a in roi[0]]
    hi = [min(int(b), n) for b, n in zip(roi[1], shapes[0])]
    if any(b <= a for a, b in zip(lo, hi)):
        raise ValueError(f"empty region of interest {roi}")
    from .sharding import parent_planes

    boxes = []
    for k in range(len(shapes) - 1):
        b0 = [a // b for a, b in zip(lo, brick)]
        b1 = [-(-h // b) for h, b in zip(hi, brick)]
        boxes.append((b0, b1))
        vlo = [max(a * b - 1, 0) for a, b in zip(b0, brick)]
        vhi = [min(c * b + 1, n) for c, b, n in zip(b1, brick, shapes[k])]
        taps = [parent_planes(vlo[d], vhi[d], shapes[k + 1][d]) for d in range(nd)]
        lo, hi = [t[0] for t in taps], [t[1] for t in taps]
    boxes.append(None)
    return boxes


def _box_list(box, grid, device):
    b0, b1 = box
    axes = [torch.arange(a, b, dtype=torch.int64) for a, b in zip(b0, b1)]
    ids = torch.zeros([len(x) for x in axes], dtype=torch.int64)
    for d, ax in enumerate(axes):
        ids = ids * grid[d] + ax.reshape([-1 if i == d else 1 for i in range(len(axes))])
    return ids.reshape(-1).to(torch.int32).to(device)


def hierarchical_random_walker(volume: torch.Tensor, seeds: torch.Tensor, brick, levels: int | None = None,
                               cfg: RWConfig = RWConfig(), *, want_labels: bool = True,
                               workspace: Workspace | None = None, level0_chunks: int | None = None,
                               on_level0_chunk=None, pyramid_store=None, pyramid_key=None,
                               roi=None) -> HRWResult:
    """Coarse-to-fine random walker (oracle/rw.py: hierarchical_random_walker).

    The coarsest level is solved whole; each finer level is initialised and
    bounded by the upsampled solution of the level above and solved brick
    by brick (multi-GPU: sharding.hierarchical_random_walker_sharded).
    `level0_chunks` > 1 solves level 0 as that many slabs of brick rows (same
    results: bricks are independent; on brick-resident levels slab c+1's system
    is built while slab c solves; default: 8 slabs for levels of >= 4096 bricks,
    else 1) and calls `on_level0_chunk(r0, r1)` after
    each with the level's (partially written) prob / labels tensors, so a
    caller can download finished rows while the rest solves.
    `roi` = (lo, hi) in level-0 voxels: solve only the bricks that region needs on every level
    (`roi_brick_boxes`); values inside it are those of the full solve, bit for bit, and NaN (labels
    255) wherever a level was not solved.
    """
    brick = tuple(int(b) for b in brick)
    if pyramid_store is not None and pyramid_key is not None:
        vols = _cached_lod_chain(volume, brick, levels, pyramid_store, pyramid_key)
    else:
        vols = lod_chain(volume, brick, levels)
    seed_levels = [seeds]
    for _ in range(len(vols) - 1):
        seed_levels.append(project_seeds(seed_levels[-1]))
    workspace = workspace or Workspace(volume.device)
    nlev = len(vols)
    probs = [None] * nlev
    stats = [None] * nlev
    top = nlev - 1
    lab = None
    top_labels = torch.empty(vols[top].shape, dtype=torch.uint8, device=volume.device) \
        if (want_labels and top == 0) else None
    # stats land in pinned host memory without host synchronisation: the whole hierarchy is
    # queued back to back, and the stats are read once at the end
    probs[top], stats[top] = solve_level(vols[top], seed_levels[top], tuple(vols[top].shape), None, cfg,
                                         labels_out=top_labels, workspace=workspace, stats_on_device=True)
    lab = top_labels
    if top == 0 and on_level0_chunk is not None:  # single-level hierarchy: level 0 is the whole-level solve
        on_level0_chunk(0, vols[0].shape[0], probs[0], top_labels)
    boxes = roi_brick_boxes([tuple(v.shape) for v in vols], brick, roi) if roi is not None else None
    skipped = [None] * nlev
    for k in range(top - 1, -1, -1):
        if boxes is not None:  # region-limited: the listed bricks, bound upsampled over their planes
            b0, b1 = boxes[k]
            grid = brick_grid(vols[k].shape, brick)
            bl = _box_list(boxes[k], grid, volume.device)
            z0, z1 = max(b0[0] * brick[0] - 1, 0), min(b1[0] * brick[0] + 1, vols[k].shape[0])
            x = upsample_planes(probs[k + 1], 0, vols[k].shape, z0, z1,
                                torch.empty(vols[k].shape, dtype=torch.float32, device=volume.device))
            out = torch.full(vols[k].shape, float("nan"), dtype=torch.float32, device=volume.device)
            lab_k = torch.full(vols[k].shape, 255, dtype=torch.uint8, device=volume.device) \
                if (want_labels and k == 0) else None
            probs[k], stats[k] = solve_level(vols[k], seed_levels[k], brick, x, cfg, brick_list=bl, out=out,
                                             labels_out=lab_k, workspace=workspace, stats_on_device=True)
            if k == 0:
                lab = lab_k
                if on_level0_chunk is not None:
                    on_level0_chunk(0, vols[0].shape[0], probs[0], lab_k)
            del x
            continue
        if cfg.skip_eps is not None:  # brick-skip rule: decided bricks keep the upsampled parent
            probs[k], stats[k], skipped[k] = _solve_level_skipping(vols[k], seed_levels[k], brick, probs[k + 1],
                                                                   cfg, want_labels and k == 0, workspace)
            if k == 0:
                lab = probs[0].gt(0.5).to(torch.uint8) if want_labels else None
                if on_level0_chunk is not None:
                    on_level0_chunk(0, vols[0].shape[0], probs[0], lab)
            continue
        if k == 0 and level0_chunks is None:  # measured: 8 slabs at 32768 bricks, 2 at 4096
            nb0 = math.prod(brick_grid(vols[0].shape, brick))
            level0_chunks = 8 if nb0 >= 16384 else (2 if nb0 >= 4096 else 1)
        # finer levels with many bricks are solved in slabs too (slab c+1's system is built while
        # slab c solves); only level 0 reports its slabs to on_level0_chunk
        nchunks = level0_chunks if k == 0 else (2 if math.prod(brick_grid(vols[k].shape, brick)) >= 4096 else 1)
        slabbed = nchunks > 1 and _resident_geometry(vols[k].shape, brick)
        x = None if slabbed else upsample(probs[k + 1], vols[k].shape)  # slabbed: upsampled slab by slab
        lab_k = torch.empty(vols[k].shape, dtype=torch.uint8, device=volume.device) \
            if (want_labels and k == 0) else None
        # separate output: the brick-resident solver reads neighbour bounds while
        # other bricks already write their results
        if slabbed:
            probs[k], stats[k] = _solve_level_chunked(vols[k], seed_levels[k], brick, probs[k + 1], cfg, lab_k,
                                                      workspace, nchunks, on_level0_chunk if k == 0 else None)
        else:
            probs[k], stats[k] = solve_level(vols[k], seed_levels[k], brick, x, cfg, labels_out=lab_k,
                                             workspace=workspace, stats_on_device=True)
            if k == 0 and on_level0_chunk is not None:
                on_level0_chunk(0, vols[0].shape[0], probs[0], lab_k)
        del x
        if k == 0:
            lab = lab_k
    if volume.is_cuda:
        torch.cuda.current_stream().synchronize()
    stats = [_merge_stats(s) if isinstance(s, list) else _resolve(s) for s in stats]
    for k, n in enumerate(skipped):
        if n is not None:
            stats[k] = dict(stats[k], skipped=n)
    return HRWResult(probs[0], lab, probs, vols, seed_levels, stats)
