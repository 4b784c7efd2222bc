"""Chunked tensor files (PLCT) streamed through the GPU — SURVEY.md §8(f)2.

The reference's on-disk format (`pkg/src/chunkcast/tensorfile.py:1-13`), restated; every field
little-endian, one tensor per file:

    magic "PLCT" | version u32 (= 1) | element code u8 | lanes u8 | ndim u8
    size ndim*u64 | chunk_size ndim*u64 | spacing ndim*f64
    offset table num_chunks*u64 (row-major chunk order, 0 = chunk absent)
    chunk payloads (each prod(chunk_size) * element width bytes, zero-padded border chunks)

Element codes (`model.py:24-29`): 0 u8, 1 i16, 2 u16, 3 f32, 4 f64; width = scalar width × lanes,
lanes innermost in a payload (`model.py:78-80`).  A pyramid is one file per level plus a JSON
manifest (`tensorfile.py:265-301`).

Where the reference resolves one chunk per positioned read into a host array
(`open_chunked`, `tensorfile.py:172-210`) and writes one chunk per call (`_ChunkWriter`,
`:108-146`), this module moves whole runs of file-contiguous chunks: disk → pinned host buffer
(one `preadv`) → device staging (async copy) → `rwb_chunks_scatter` into the dense level tensor,
double-buffered so the next run is read while the previous one is copied and scattered; saving
is the mirror image (`rwb_chunks_gather` → device-to-host copy → one `write` per run).  Files
written here are byte-identical to the reference writer's for the same tensor (chunks in
row-major order, the offset table of `import_raw`).  `build_lod_offline` materialises the LOD
pyramid of a file with the GPU LOD kernel (`tensorfile.py:307-341`), and `segment_file` runs the
hierarchical random walker from files to files.
"""

from __future__ import annotations

import json
import math
import os
import struct
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
import torch

from . import _native, device

MAGIC = b"PLCT"
VERSION = 1
_FIXED = struct.Struct("<4sIBBB")

# code -> (label, numpy dtype, torch dtype)
SCALARS = {
    0: ("u8", np.dtype("<u1"), torch.uint8),
    1: ("i16", np.dtype("<i2"), torch.int16),
    2: ("u16", np.dtype("<u2"), torch.uint16),
    3: ("f32", np.dtype("<f4"), torch.float32),
    4: ("f64", np.dtype("<f8"), torch.float64),
}
_CODE_OF = {v[2]: k for k, v in SCALARS.items()}


class PlctError(OSError):
    """Malformed or unsupported chunked tensor file (the reference's TensorFileError)."""


@dataclass(frozen=True)
class Header:
    size: tuple
    chunk: tuple
    code: int
    lanes: int
    spacing: tuple
    offsets: np.ndarray  # u64 per chunk, row-major; 0 = absent
    header_bytes: int

    @property
    def ndim(self) -> int:
        return len(self.size)

    @property
    def grid(self) -> tuple:
        return tuple(-(-s // c) for s, c in zip(self.size, self.chunk))

    @property
    def num_chunks(self) -> int:
        return math.prod(self.grid)

    @property
    def elem_bytes(self) -> int:
        return SCALARS[self.code][1].itemsize * self.lanes

    @property
    def payload_bytes(self) -> int:
        return math.prod(self.chunk) * self.elem_bytes

    @property
    def torch_dtype(self):
        return SCALARS[self.code][2]

    @property
    def dense_shape(self) -> tuple:
        return tuple(self.size) + ((self.lanes,) if self.lanes > 1 else ())


def header_size(ndim: int, num_chunks: int) -> int:
    return _FIXED.size + ndim * 8 * 3 + num_chunks * 8


def _pack_header(size, chunk, code, lanes, spacing, offsets) -> bytes:
    nd = len(size)
    return b"".join([
        _FIXED.pack(MAGIC, VERSION, code, lanes, nd),
        struct.pack(f"<{nd}Q", *[int(s) for s in size]),
        struct.pack(f"<{nd}Q", *[int(c) for c in chunk]),
        struct.pack(f"<{nd}d", *[float(s) for s in spacing]),
        np.asarray(offsets, dtype="<u8").tobytes(),
    ])


def read_header(path) -> Header:
    """Parse and validate a chunked file's header and offset table (`tensorfile.py:63-91`)."""
    path = os.fspath(path)
    file_size = os.path.getsize(path)
    with open(path, "rb") as f:
        def exact(n):
            b = f.read(n)
            if len(b) != n:
                raise PlctError(f"{path}: truncated file")
            return b

        magic, version, code, lanes, nd = _FIXED.unpack(exact(_FIXED.size))
        if magic != MAGIC:
            raise PlctError(f"{path}: not a chunked tensor file (bad magic)")
        if version != VERSION:
            raise PlctError(f"{path}: unsupported version {version}")
        if code not in SCALARS:
            raise PlctError(f"{path}: unknown scalar code {code}")
        if not 1 <= lanes <= 4:
            raise PlctError(f"{path}: lanes must be 1-4, got {lanes}")
        size = struct.unpack(f"<{nd}Q", exact(nd * 8))
        chunk = struct.unpack(f"<{nd}Q", exact(nd * 8))
        spacing = struct.unpack(f"<{nd}d", exact(nd * 8))
        if any(s < 1 for s in size) or any(c < 1 for c in chunk):
            raise PlctError(f"{path}: sizes and chunk sizes must be positive")
        n = math.prod(-(-s // c) for s, c in zip(size, chunk))
        offsets = np.frombuffer(exact(n * 8), dtype="<u8").copy()
    hb = header_size(nd, n)
    h = Header(tuple(size), tuple(chunk), code, lanes, tuple(spacing), offsets, hb)
    present = offsets[offsets != 0]
    if present.size and (present.min() < hb or present.max() + h.payload_bytes > file_size):
        raise PlctError(f"{path}: chunk offset outside file")
    return h


# file I/O of a run is split over a few threads (os.preadv / os.pwrite release the GIL): one
# thread copying out of the page cache tops out near 6 GB/s, far below PCIe
_IO_THREADS = max(1, min(8, len(os.sched_getaffinity(0))))
_io_pool = None


def _pool():
    global _io_pool
    if _io_pool is None:
        _io_pool = ThreadPoolExecutor(_IO_THREADS, thread_name_prefix="plct-io")
    return _io_pool


def _parallel_io(fn, fd, view: np.ndarray, offset: int, what: str) -> None:
    """Read (`os.preadv`) or write (`os.pwrite`) `view` at file `offset` in parallel parts."""
    n = view.nbytes
    parts = max(1, min(_IO_THREADS, n >> 22))  # >= 4 MiB per part
    step = -(-n // parts)

    def one(k):
        a, b = k * step, min(n, (k + 1) * step)
        mv = memoryview(view)[a:b]
        done = 0
        while done < b - a:
            got = fn(fd, mv[done:], offset + a + done)
            if got <= 0:
                raise PlctError(f"short {what} at byte {offset + a + done}")
            done += got

    list(_pool().map(one, range(parts)))


def _preadv1(fd, mv, off):
    return os.preadv(fd, [mv], off)


class _Staging:
    """Two pinned host buffers and two device buffers of `nbytes` for double-buffered transfers."""

    def __init__(self, nbytes: int, dev: torch.device):
        self.host = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
        self.dev = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
        self.done = [None, None]  # event after the last use of buffer pair b

    def wait(self, b):
        if self.done[b] is not None:
            self.done[b].synchronize()


def _runs(ids_by_offset, offsets, payload, max_chunks):
    """Split chunk ids (sorted by file offset) into runs that are contiguous in the file."""
    run = []
    for cid in ids_by_offset:
        if run and (len(run) == max_chunks or offsets[cid] != offsets[run[-1]] + payload):
            yield run
            run = []
        run.append(cid)
    if run:
        yield run


def _ids_arg(run, dev, keep):
    """(chunk_ids device pointer or None, first) for a run of chunk ids."""
    if all(b == a + 1 for a, b in zip(run, run[1:])):
        return None, int(run[0])
    ids_h = torch.tensor(run, dtype=torch.int64).pin_memory()
    ids_d = ids_h.to(dev, non_blocking=True)
    keep.extend([ids_h, ids_d])
    return ids_d.data_ptr(), 0


def load(path, device_=None, *, staging_bytes: int = 64 << 20) -> tuple:
    """Read a chunked file into a dense device tensor; returns (tensor, Header).

    Absent chunks read as zeros (`open_chunked`, `tensorfile.py:186-190`).  The tensor is
    complete in stream order on the current stream when this returns.
    """
    path = os.fspath(path)
    h = read_header(path)
    dev = torch.device(device_) if device_ is not None else torch.device("cuda", torch.cuda.current_device())
    lib = _native.lib()
    out = torch.empty(h.dense_shape, dtype=h.torch_dtype, device=dev)
    present = np.flatnonzero(h.offsets)
    if present.size < h.num_chunks:
        out.view(torch.uint8).zero_()
    if present.size == 0:
        return out, h
    P = h.payload_bytes
    per = max(1, min(staging_bytes // P, present.size))
    stg = _Staging(per * P, dev)
    size_a, chunk_a = _native.int64_array(h.size), _native.int64_array(h.chunk)
    comp = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)
    side.wait_stream(comp)  # `out` (and its zeroing) before the scatters
    keep = []
    order = present[np.argsort(h.offsets[present], kind="stable")]
    fd = os.open(path, os.O_RDONLY)
    try:
        for i, run in enumerate(_runs(order.tolist(), h.offsets, P, per)):
            b = i & 1
            stg.wait(b)
            nbytes = len(run) * P
            view = stg.host[b].numpy()[:nbytes]
            _parallel_io(_preadv1, fd, view, int(h.offsets[run[0]]), f"read of {path}")
            with torch.cuda.stream(side):
                stg.dev[b][:nbytes].copy_(stg.host[b][:nbytes], non_blocking=True)
                ids, first = _ids_arg(run, dev, keep)
                _native.check(lib.rwb_chunks_scatter(h.ndim, size_a, chunk_a, h.elem_bytes, stg.dev[b].data_ptr(),
                                                     ids, first, len(run), out.data_ptr(), side.cuda_stream))
                ev = torch.cuda.Event()
                ev.record(side)
                stg.done[b] = ev
    finally:
        os.close(fd)
    comp.wait_stream(side)
    for t in keep + stg.dev:  # device buffers stay reserved until the scatters ran (pinned host ones
        if t.is_cuda:          # are tracked by torch's host allocator)
            t.record_stream(comp)
    return out, h


def _element_of(t: torch.Tensor, lanes: int):
    if t.dtype not in _CODE_OF:
        raise ValueError(f"unsupported dtype {t.dtype} (u8, i16, u16, f32, f64)")
    return _CODE_OF[t.dtype], lanes


def save(tensor: torch.Tensor, path, chunk, spacing=None, *, lanes: int = 1,
         staging_bytes: int = 64 << 20) -> Header:
    """Write a dense device tensor as a chunked file (every chunk present, row-major order, the
    layout `import_raw` / `save_tensor` produce, `tensorfile.py:149-165, 213-219`)."""
    path = os.fspath(path)
    if not tensor.is_cuda:
        raise ValueError("save: tensor must be a CUDA tensor")
    t = tensor.contiguous()
    size = tuple(int(s) for s in (t.shape[:-1] if lanes > 1 else t.shape))
    if lanes > 1 and t.shape[-1] != lanes:
        raise ValueError(f"save: last dimension {t.shape[-1]} is not lanes={lanes}")
    chunk = tuple(int(c) for c in chunk)
    if len(chunk) != len(size):
        raise ValueError("save: chunk rank differs from the tensor's")
    spacing = tuple(float(s) for s in (spacing if spacing is not None else (1.0,) * len(size)))
    code, lanes = _element_of(t, lanes)
    grid = tuple(-(-s // c) for s, c in zip(size, chunk))
    n = math.prod(grid)
    eb = SCALARS[code][1].itemsize * lanes
    P = math.prod(chunk) * eb
    hb = header_size(len(size), n)
    offsets = hb + P * np.arange(n, dtype=np.uint64)
    lib = _native.lib()
    dev = t.device
    per = max(1, min(staging_bytes // P, n))
    stg = _Staging(per * P, dev)
    size_a, chunk_a = _native.int64_array(size), _native.int64_array(chunk)
    comp = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)
    side.wait_stream(comp)  # the tensor is complete before the gathers
    pending = None  # (buffer, nbytes, file offset) copied to the host, not yet written
    fd = os.open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
    try:
        try:  # the file's blocks up front: the parallel writes then only fill pages
            os.posix_fallocate(fd, 0, hb + n * P)
        except OSError:
            pass
        head = _pack_header(size, chunk, code, lanes, spacing, offsets)
        _parallel_io(os.pwrite, fd, np.frombuffer(head, dtype=np.uint8), 0, f"write of {path}")
        for i, first in enumerate(range(0, n, per)):
            b = i & 1
            cnt = min(per, n - first)
            stg.wait(b)  # its bytes were written below before this buffer comes round again
            with torch.cuda.stream(side):
                _native.check(lib.rwb_chunks_gather(len(size), size_a, chunk_a, eb, t.data_ptr(), None, first, cnt,
                                                    stg.dev[b].data_ptr(), side.cuda_stream))
                stg.host[b][:cnt * P].copy_(stg.dev[b][:cnt * P], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
                stg.done[b] = ev
            if pending is not None:
                pb, pn, po = pending
                stg.wait(pb)
                _parallel_io(os.pwrite, fd, stg.host[pb].numpy()[:pn], po, f"write of {path}")
            pending = (b, cnt * P, hb + first * P)
        if pending is not None:
            pb, pn, po = pending
            stg.wait(pb)
            _parallel_io(os.pwrite, fd, stg.host[pb].numpy()[:pn], po, f"write of {path}")
    finally:
        os.close(fd)
    t.record_stream(side)
    return read_header(path)


# ---------------------------------------------------------------------------
# pyramid manifests (tensorfile.py:226-301)


@dataclass(frozen=True)
class PyramidLevel:
    path: str
    spacing: tuple
    const_table: str | None = None


def save_manifest(levels, path) -> None:
    path = os.fspath(path)
    base = os.path.dirname(os.path.abspath(path))
    doc = {
        "format": "chunked-pyramid",
        "version": 1,
        "levels": [{
            "path": os.path.relpath(lv.path, base),
            "spacing": [float(s) for s in lv.spacing],
            "const_table": os.path.relpath(lv.const_table, base) if lv.const_table else None,
        } for lv in levels],
    }
    with open(path, "w", encoding="utf-8") as f:
        json.dump(doc, f, indent=2, sort_keys=True)
        f.write("\n")


def load_manifest(path) -> tuple:
    path = os.fspath(path)
    try:
        with open(path, encoding="utf-8") as f:
            doc = json.load(f)
    except json.JSONDecodeError as exc:
        raise PlctError(f"{path}: not a manifest: {exc}") from None
    if doc.get("format") != "chunked-pyramid":
        raise PlctError(f"{path}: not a pyramid manifest")
    base = os.path.dirname(os.path.abspath(path))

    def absolute(p):
        return p if p is None or os.path.isabs(p) else os.path.join(base, p)

    levels = tuple(PyramidLevel(absolute(lv["path"]), tuple(lv["spacing"]), absolute(lv.get("const_table")))
                   for lv in doc["levels"])
    if not levels:
        raise PlctError("manifest has no levels")
    return levels


def const_chunk_table(level: torch.Tensor, chunk) -> torch.Tensor:
    """Per-chunk uniform value or sentinel (NaN / type max) over the chunk grid of a scalar device
    tensor (`build_const_chunk_table`, ops.py:777-816), on the GPU."""
    if level.dtype not in _CODE_OF:
        raise ValueError(f"unsupported dtype {level.dtype}")
    t = level.contiguous()
    grid = tuple(-(-int(s) // int(c)) for s, c in zip(t.shape, chunk))
    out = torch.empty(grid, dtype=t.dtype, device=t.device)
    _native.check(_native.lib().rwb_const_chunk_table(t.dim(), _native.int64_array(t.shape), _native.int64_array(chunk),
                                                      _CODE_OF[t.dtype], t.data_ptr(), out.data_ptr(),
                                                      torch.cuda.current_stream(t.device).cuda_stream))
    return out


def _save_const_table(level, chunk, path):
    table = const_chunk_table(level, chunk)
    tchunk = tuple(min(int(c), int(g)) for c, g in zip(chunk, table.shape))  # ops.py:787-788
    save(table, path, tchunk, None)


def build_lod_offline(input_path, manifest_path, *, smooth: bool = True, const_tables: bool = False) -> tuple:
    """Materialise the LOD pyramid of a chunked f32 file (`tensorfile.py:307-341`).

    Level 0 is the input file itself; level k+1 = f32(downsample_mean(separable_conv(level k)))
    (or downsample_mean alone when `smooth` is False) computed on the GPU — bit-identical to the
    reference's operators — and saved as `<manifest base>.L<k+1>.plct` with the same chunk size
    and doubled spacing, until every dimension fits one chunk.  `const_tables` also writes each
    level's constant-chunk table as `<base>.L<k>.ctab.plct`.  Returns the manifest's levels.
    """
    input_path = os.path.abspath(os.fspath(input_path))
    manifest_path = os.fspath(manifest_path)
    base = os.path.splitext(os.path.abspath(manifest_path))[0]
    level, h = load(input_path)
    if h.code != 3 or h.lanes != 1 or h.ndim > 3:
        raise ValueError("build_lod_offline: the GPU LOD kernels take 1- to 3-D f32 scalar tensors")
    def table(lv, k):  # the level's constant-chunk table file, when asked for
        if not const_tables:
            return None
        ct = f"{base}.L{k}.ctab.plct"
        _save_const_table(lv, h.chunk, ct)
        return ct

    levels = [PyramidLevel(input_path, h.spacing, table(level, 0))]
    size, spacing, k = h.size, h.spacing, 0
    while not all(s <= c for s, c in zip(size, h.chunk)):
        level = device.lod_down(level) if smooth else device.downsample_mean(level)
        spacing = tuple(2.0 * s for s in spacing)
        size = tuple(level.shape)
        path = f"{base}.L{k + 1}.plct"
        save(level, path, h.chunk, spacing)
        k += 1
        levels.append(PyramidLevel(path, spacing, table(level, k)))
    save_manifest(levels, manifest_path)
    return tuple(levels)


def segment_file(volume_path, seeds_path, prob_path, labels_path=None, brick=None, levels=None, cfg=None, *,
                 workspace=None):
    """Hierarchical random walker from chunked files to chunked files.

    The f32 volume and u8 seeds stream from disk to the device, the hierarchy runs there, and the
    probabilities (f32) and labels (u8) stream back to new files with the volume's chunk size and
    spacing.  `brick` defaults to the file's chunk size.  Returns the solver's HRWResult.
    """
    from .config import RWConfig

    vol, hv = load(volume_path)
    seeds, hs = load(seeds_path)
    if hv.code != 3 or hs.code != 0 or hv.lanes != 1 or hs.lanes != 1 or hv.size != hs.size:
        raise ValueError("segment_file: expects an f32 volume and u8 seeds of the same size")
    brick = tuple(brick) if brick is not None else hv.chunk
    res = device.hierarchical_random_walker(vol, seeds, brick, levels, cfg or RWConfig(), workspace=workspace)
    save(res.prob, prob_path, hv.chunk, hv.spacing)
    if labels_path is not None:
        save(res.labels, labels_path, hv.chunk, hv.spacing)
    return res
