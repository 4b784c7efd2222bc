"""HBM chunk store with a byte budget — SURVEY.md §8(f)1.

The reference's bounded chunk store (`pkg/src/chunkcast/store.py:145-342`), restated for device
memory: every allocation is a slab of HBM (a CUDA `uint8` tensor), so level slabs, chunk
payloads and results can stay resident on the GPU under a fixed budget and be evicted LRU-first
when it runs out.  Semantics kept from the reference:

* sizes are quantised to buckets of at most `mantissa_bits` significant bits below the leading
  one (`quantize_size`, `:73-83`); freed allocations park in a per-size bucket cache and are
  handed back to the next allocation of the same quantised size (`:170-205`), and occupancy
  counts live entries plus cached buckets, so the capacity is a hard bound on owned HBM;
* entries carry a state (IN_FLIGHT < PREVIEW < FINAL, `:67-70`); a duplicate insert keeps the
  stronger state (`:217-246`); lookups pin, unpins re-queue for LRU (`:261-287`);
* garbage collection pops the LRU queue until `gc_target_fraction * capacity` bytes are freed
  and stops early at the first entry whose epoch has not completed (`:335-362`); here an epoch is
  a CUDA event recorded on the stream that produced the entry, so a payload is never recycled
  while a kernel may still be writing or reading it.  When the sweep falls short, the bucket
  cache is flushed back to the CUDA allocator.

`put(id, tensor)` / `get(id, dtype, shape)` are the typed conveniences on top (device-to-device
copy in, a tensor view out).
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass
from enum import IntEnum

import torch


class StoreError(Exception):
    pass


class AllocationTooLarge(StoreError):
    """Requested size exceeds the store's capacity; retrying cannot help."""


class ReclamationNeeded(StoreError):
    """Capacity exhausted; run garbage_collect() and retry."""


class ChunkState(IntEnum):
    IN_FLIGHT = 0
    PREVIEW = 1
    FINAL = 2


def quantize_size(requested: int, mantissa_bits: int = 8) -> int:
    """Round a byte size up to its bucket: granularity 2^max(0, floor(log2 s) - mantissa_bits)."""
    if requested < 1:
        raise ValueError("size must be positive")
    g = 1 << max(0, requested.bit_length() - 1 - mantissa_bits)
    return -(-requested // g) * g


@dataclass
class Allocation:
    size_q: int
    buffer: torch.Tensor | None  # uint8 CUDA tensor of size_q bytes


@dataclass
class Entry:
    id: object
    size_bytes: int
    size_q: int
    state: ChunkState
    lru_stamp: int
    epoch: int
    allocation: Allocation | None
    ref_count: int = 0

    @property
    def payload(self) -> torch.Tensor:
        return self.allocation.buffer[: self.size_bytes]


class DeviceStore:
    """Bounded HBM store at one device (the reference's `Store` with device buffers)."""

    def __init__(self, capacity: int, device=None, *, gc_target_fraction: float = 0.10, mantissa_bits: int = 8):
        if not 0 < gc_target_fraction <= 1:
            raise ValueError("gc_target_fraction must be in (0, 1]")
        self.capacity = int(capacity)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.gc_target_fraction = gc_target_fraction
        self.mantissa_bits = mantissa_bits
        self.entries: dict = {}
        self.live_bytes = 0
        self.cached_bytes = 0
        self.buckets: dict[int, list[Allocation]] = {}
        self.evictions = 0
        self._heap: list = []
        self._seq = 0
        self._stamp = 0
        self._events: list = []  # (epoch, event), epochs ascending
        self.current_epoch = 0
        self.completed_epoch = 0

    # -- epochs ---------------------------------------------------------------------------

    def record_epoch(self, stream=None) -> int:
        """Close an epoch on `stream` (default: current): entries inserted with it become
        collectable once the stream has passed this point."""
        self.current_epoch += 1
        ev = torch.cuda.Event()
        ev.record(stream if stream is not None else torch.cuda.current_stream(self.device))
        self._events.append((self.current_epoch, ev))
        return self.current_epoch

    def poll_epochs(self) -> int:
        """Advance completed_epoch over the events that have completed, in order."""
        while self._events and self._events[0][1].query():
            self.completed_epoch = self._events.pop(0)[0]
        return self.completed_epoch

    # -- allocation -----------------------------------------------------------------------

    def allocate(self, size_bytes: int) -> Allocation:
        size_q = quantize_size(int(size_bytes), self.mantissa_bits)
        if size_q > self.capacity:
            raise AllocationTooLarge(f"allocation of {size_bytes} bytes exceeds the capacity {self.capacity}")
        bucket = self.buckets.get(size_q)
        if bucket:
            alloc = bucket.pop()
            self.cached_bytes -= size_q
            self.live_bytes += size_q
            return alloc
        if self.live_bytes + self.cached_bytes + size_q > self.capacity:
            raise ReclamationNeeded(f"device store full ({self.occupancy()}/{self.capacity})")
        alloc = Allocation(size_q, torch.empty(size_q, dtype=torch.uint8, device=self.device))
        self.live_bytes += size_q
        return alloc

    def free_allocation(self, alloc: Allocation) -> None:
        self.live_bytes -= alloc.size_q
        self.cached_bytes += alloc.size_q
        self.buckets.setdefault(alloc.size_q, []).append(alloc)

    def flush_buckets(self) -> int:
        freed = self.cached_bytes
        for allocs in self.buckets.values():
            for a in allocs:
                a.buffer = None  # back to the CUDA caching allocator
        self.buckets.clear()
        self.cached_bytes = 0
        return freed

    def occupancy(self) -> int:
        return self.live_bytes + self.cached_bytes

    # -- entries --------------------------------------------------------------------------

    def _next_stamp(self) -> int:
        self._stamp += 1
        return self._stamp

    def _lru_push(self, e: Entry) -> None:
        self._seq += 1
        heapq.heappush(self._heap, (e.lru_stamp, self._seq, e.id))

    def insert(self, id, alloc: Allocation, nbytes: int, state: ChunkState = ChunkState.FINAL,
               epoch: int | None = None) -> Entry:
        """Register bytes written into `alloc` (by work queued on the current stream) under `id`;
        `epoch` defaults to a new one recorded now."""
        existing = self.entries.get(id)
        if existing is not None and existing.state >= state and existing.state != ChunkState.IN_FLIGHT:
            self.free_allocation(alloc)
            return existing
        if existing is not None:
            self._drop(existing, recycle=existing.ref_count == 0)
        e = Entry(id, int(nbytes), alloc.size_q, ChunkState(state), self._next_stamp(),
                  self.record_epoch() if epoch is None else int(epoch), alloc)
        self.entries[id] = e
        self._lru_push(e)
        return e

    def _drop(self, e: Entry, recycle: bool) -> None:
        del self.entries[e.id]
        if recycle:
            self.free_allocation(e.allocation)
        else:  # a reader still holds the payload; the bytes leave the store's accounting
            self.live_bytes -= e.size_q
        e.allocation = None

    def lookup(self, id, min_state: ChunkState = ChunkState.FINAL) -> Entry | None:
        """The entry, pinned, if present at `min_state` or stronger (never IN_FLIGHT)."""
        e = self.entries.get(id)
        if e is None or e.state < min_state or e.state == ChunkState.IN_FLIGHT:
            return None
        e.ref_count += 1
        e.lru_stamp = self._next_stamp()
        return e

    def unpin(self, e: Entry) -> None:
        if e.ref_count <= 0:
            raise StoreError("unbalanced unpin")
        e.ref_count -= 1
        if e.ref_count == 0 and self.entries.get(e.id) is e:
            self._lru_push(e)

    def garbage_collect(self, target_bytes: int | None = None) -> int:
        """Evict unpinned entries LRU-first until `target_bytes` (default gc_target_fraction x
        capacity) are freed, stopping at the first entry whose epoch is still running."""
        completed = self.poll_epochs()
        if target_bytes is None:
            target_bytes = int(self.gc_target_fraction * self.capacity)
        freed = 0
        while freed < target_bytes and self._heap:
            stamp, _, id = self._heap[0]
            e = self.entries.get(id)
            if e is None or e.ref_count > 0 or e.lru_stamp != stamp:
                heapq.heappop(self._heap)  # stale
                continue
            if e.epoch > completed:
                break
            heapq.heappop(self._heap)
            self._drop(e, recycle=True)
            self.evictions += 1
            freed += e.size_q
        if freed < target_bytes:
            self.flush_buckets()
        return freed

    # -- typed conveniences ---------------------------------------------------------------

    def put(self, id, tensor: torch.Tensor, state: ChunkState = ChunkState.FINAL) -> Entry:
        """Copy a device tensor into the store (collecting garbage once if the budget is full)."""
        t = tensor.contiguous()
        nbytes = t.numel() * t.element_size()
        try:
            alloc = self.allocate(nbytes)
        except ReclamationNeeded:
            self.garbage_collect(max(quantize_size(nbytes, self.mantissa_bits),
                                     int(self.gc_target_fraction * self.capacity)))
            alloc = self.allocate(nbytes)
        alloc.buffer[:nbytes].copy_(t.view(-1).view(torch.uint8), non_blocking=True)
        return self.insert(id, alloc, nbytes, state)

    def get(self, id, dtype, shape, min_state: ChunkState = ChunkState.FINAL):
        """(pinned entry, typed view of its payload) or None; unpin the entry when done."""
        e = self.lookup(id, min_state)
        if e is None:
            return None
        return e, e.payload.view(dtype).view(shape)
