"""HBM chunk store: ONE device arena under a hard byte budget — SURVEY.md §8(f)1.

The reference keeps chunks in a bounded store with size-quantised free buckets, LRU eviction and
epoch-gated garbage collection (`pkg/src/chunkcast/store.py:73-83, 145-362`); Palace allocates its
bounded memory regions once at start-up (`PAPER.md:207-209`).  On the GPU that becomes:

* **one allocation**: the store reserves `capacity` bytes of HBM at construction
  (`torch.empty(capacity, uint8)`) and never calls the CUDA allocator again.  Payloads are
  extents (offset, length) of that arena; a best-fit free list keeps extents sorted by address
  and merges neighbours when they are returned, so the arena fragments as little as the
  allocation pattern allows.
* **the reference's accounting, unchanged**: requests are rounded to their `quantize_size` bucket
  (at most `mantissa_bits` significant bits below the leading one); freed extents first park in
  a per-bucket cache and serve the next request of the same bucket; occupancy = live + parked
  bytes <= capacity; a duplicate insert keeps the stronger state (IN_FLIGHT < PREVIEW < FINAL);
  lookups pin and refresh the LRU stamp; `garbage_collect` evicts unpinned entries LRU-first
  until the target is freed and stops at the first entry whose epoch is still running, then
  returns the parked extents to the arena when it fell short.  `tests/test_store.py` drives
  the reference `Store` and this one with the same random operation sequences (shadow model).
* **stream-ordered reuse**: an epoch is a CUDA event recorded on the stream that produced or last
  read an entry (`retire`); an extent parked while a kernel may still touch it carries the epoch
  of its release and is handed out again only once that event has completed, so recycling HBM
  never races queued work.  (A CPU arena — `device="cpu"` — completes every epoch at once: the
  host-side tests of the accounting.)
* **physical vs accounted bytes**: extents are 256-byte aligned.  Accounting follows the reference
  (quantised sizes); an arena that is fragmented, or whose alignment slack exceeds the accounted
  headroom, raises `ReclamationNeeded` like a full store.

`put(id, tensor)` / `get(id, dtype, shape)` are typed conveniences (device-to-device copy in, a
typed view of the payload out); `reserve(id, nbytes)` hands out an IN_FLIGHT entry to be written
by queued work and published with `publish` (used by `api.segment_series` to stream a 4-D series
through a budget below its size).
"""

from __future__ import annotations

import bisect
import heapq
from dataclasses import dataclass
from enum import IntEnum

import torch

ALIGN = 256


class StoreError(Exception):
    pass


class AllocationTooLarge(StoreError):
    """Requested size exceeds the store's capacity; retrying cannot help."""


class ReclamationNeeded(StoreError):
    """Capacity (or a contiguous extent) exhausted; run garbage_collect() and retry."""


class ChunkState(IntEnum):
    IN_FLIGHT = 0
    PREVIEW = 1
    FINAL = 2


def quantize_size(requested: int, mantissa_bits: int = 8) -> int:
    """Bucket of a byte size: keep `mantissa_bits` significant bits below the leading one, round up
    (the reference rule, `store.py:73-83`; overshoot below 1/256 for the default)."""
    if requested < 1:
        raise ValueError("size must be positive")
    step = 1 << max(0, requested.bit_length() - 1 - mantissa_bits)
    return ((requested + step - 1) // step) * step


def _aligned(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


class Arena:
    """Best-fit extent allocator over one buffer; free extents sorted by offset, merged on release."""

    def __init__(self, nbytes: int, device):
        self.nbytes = int(nbytes)
        self.buffer = torch.empty(self.nbytes, dtype=torch.uint8, device=device)
        self._starts = [0]          # free extents, by offset
        self._lens = [self.nbytes]

    def take(self, length: int) -> int | None:
        best = -1
        for k, n in enumerate(self._lens):
            if n >= length and (best < 0 or n < self._lens[best]):
                best = k
                if n == length:
                    break
        if best < 0:
            return None
        off = self._starts[best]
        if self._lens[best] == length:
            del self._starts[best], self._lens[best]
        else:
            self._starts[best] += length
            self._lens[best] -= length
        return off

    def give(self, off: int, length: int) -> None:
        k = bisect.bisect_left(self._starts, off)
        self._starts.insert(k, off)
        self._lens.insert(k, length)
        if k + 1 < len(self._starts) and off + length == self._starts[k + 1]:  # merge right
            self._lens[k] += self._lens.pop(k + 1)
            self._starts.pop(k + 1)
        if k > 0 and self._starts[k - 1] + self._lens[k - 1] == off:  # merge left
            self._lens[k - 1] += self._lens.pop(k)
            self._starts.pop(k)

    def free_bytes(self) -> int:
        return sum(self._lens)

    def largest_free(self) -> int:
        return max(self._lens, default=0)


@dataclass
class Allocation:
    size_q: int          # accounted (quantised) bytes
    offset: int          # extent in the arena
    length: int          # physical bytes (aligned)
    store: "DeviceStore"
    free_epoch: int = 0  # parked: reusable once this epoch has completed

    @property
    def buffer(self) -> torch.Tensor:
        return self.store.arena.buffer[self.offset: self.offset + self.length]


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
    """Bounded HBM chunk store over one arena at one device."""

    def __init__(self, capacity: int, device=None, *, gc_target_fraction: float = 0.10, mantissa_bits: int = 8):
        if not 0 < gc_target_fraction <= 1:
            raise ValueError("gc_target_fraction must be in (0, 1]")
        self.capacity = int(capacity)
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.gc_target_fraction = gc_target_fraction
        self.mantissa_bits = mantissa_bits
        self.arena = Arena(self.capacity, self.device)
        self.entries: dict = {}
        self.live_bytes = 0
        self.cached_bytes = 0
        self.parked: dict[int, list[Allocation]] = {}  # bucket -> parked extents, oldest first
        self.evictions = 0
        self.hits = 0
        self.misses = 0
        self.peak_occupancy = 0
        self._lru: list = []   # (stamp, seq, id); stale items skipped lazily
        self._seq = 0
        self._clock = 0
        self._pending: list = []  # (epoch, event) not yet known complete, epochs ascending
        self.current_epoch = 0
        self.completed_epoch = 0

    # -- epochs ---------------------------------------------------------------------------

    def record_epoch(self, stream=None) -> int:
        """A new epoch, complete once `stream` (default: the current one) passes this point."""
        self.current_epoch += 1
        if self.device.type == "cuda":
            ev = torch.cuda.Event()
            ev.record(stream if stream is not None else torch.cuda.current_stream(self.device))
            self._pending.append((self.current_epoch, ev))
        else:
            self.completed_epoch = self.current_epoch
        return self.current_epoch

    def poll_epochs(self) -> int:
        while self._pending and self._pending[0][1].query():
            self.completed_epoch = self._pending.pop(0)[0]
        return self.completed_epoch

    def wait_epoch(self, epoch: int) -> None:
        """Block the host until `epoch` has completed."""
        while self._pending and self._pending[0][0] <= epoch:
            e, ev = self._pending.pop(0)
            ev.synchronize()
            self.completed_epoch = e

    # -- allocation -----------------------------------------------------------------------

    def allocate(self, size_bytes: int) -> Allocation:
        size_q = quantize_size(int(size_bytes), self.mantissa_bits)
        if size_q > self.capacity:
            raise AllocationTooLarge(f"allocation of {size_bytes} bytes exceeds the capacity {self.capacity}")
        parked = self.parked.get(size_q)
        if parked:
            done = self.poll_epochs() if parked[0].free_epoch > self.completed_epoch else self.completed_epoch
            if parked[0].free_epoch <= done:
                a = parked.pop(0)
                self.cached_bytes -= size_q
                self.live_bytes += size_q
                return a
        if self.live_bytes + self.cached_bytes + size_q > self.capacity:
            raise ReclamationNeeded(f"device store full ({self.occupancy()}/{self.capacity})")
        length = _aligned(size_q)
        off = self.arena.take(length)
        if off is None:
            raise ReclamationNeeded(f"no free extent of {length} bytes (largest {self.arena.largest_free()})")
        self.live_bytes += size_q
        self.peak_occupancy = max(self.peak_occupancy, self.occupancy())
        return Allocation(size_q, off, length, self)

    def free_allocation(self, alloc: Allocation, epoch: int | None = None) -> None:
        """Park the extent in its bucket; reusable once `epoch` (default: the last recorded one)
        has completed."""
        self.live_bytes -= alloc.size_q
        self.cached_bytes += alloc.size_q
        alloc.free_epoch = self.current_epoch if epoch is None else int(epoch)
        self.parked.setdefault(alloc.size_q, []).append(alloc)

    def flush_buckets(self) -> int:
        """Return every parked extent whose epoch has completed to the arena."""
        done = self.poll_epochs()
        freed = 0
        for size_q in list(self.parked):
            keep = []
            for a in self.parked[size_q]:
                if a.free_epoch <= done:
                    self.arena.give(a.offset, a.length)
                    freed += size_q
                else:
                    keep.append(a)
            if keep:
                self.parked[size_q] = keep
            else:
                del self.parked[size_q]
        self.cached_bytes -= freed
        return freed

    def occupancy(self) -> int:
        return self.live_bytes + self.cached_bytes

    # -- entries --------------------------------------------------------------------------

    def _tick(self) -> int:
        self._clock += 1
        return self._clock

    def _queue(self, e: Entry) -> None:
        self._seq += 1
        heapq.heappush(self._lru, (e.lru_stamp, self._seq, e.id))

    def insert(self, id, alloc: Allocation, nbytes: int, state: ChunkState = ChunkState.FINAL,
               epoch: int | None = None) -> Entry:
        """Publish bytes written into `alloc` (by work queued on the current stream) under `id`;
        `epoch` defaults to a new one recorded now."""
        old = self.entries.get(id)
        if old is not None and old.state != ChunkState.IN_FLIGHT and old.state >= state:
            self.free_allocation(alloc)
            return old
        if old is not None:  # replaced: its extent waits for the work queued so far
            self._remove(old, reuse=old.ref_count == 0, epoch=self.record_epoch())
        e = Entry(id, int(nbytes), alloc.size_q, ChunkState(state), self._tick(),
                  self.record_epoch() if epoch is None else int(epoch), alloc)
        self.entries[id] = e
        self._queue(e)
        return e

    def _remove(self, e: Entry, reuse: bool, epoch: int) -> None:
        del self.entries[e.id]
        if reuse:
            self.free_allocation(e.allocation, epoch)
        else:  # a reader still holds the payload: its bytes leave the accounting
            self.live_bytes -= e.size_q
        e.allocation = None

    def lookup(self, id, min_state: ChunkState = ChunkState.FINAL) -> Entry | None:
        """The entry, pinned, when present at `min_state` or stronger (never IN_FLIGHT)."""
        e = self.entries.get(id)
        if e is None or e.state == ChunkState.IN_FLIGHT or e.state < min_state:
            self.misses += 1
            return None
        self.hits += 1
        e.ref_count += 1
        e.lru_stamp = self._tick()
        return e

    def unpin(self, e: Entry) -> None:
        """Release a pin taken after queueing reads of the payload on the current stream (the
        entry is collectable once they have run; `retire` names another stream)."""
        self.retire(e)

    def retire(self, e: Entry, stream=None) -> None:
        """Unpin after queueing work that reads (or writes) the payload on `stream`: the entry
        becomes collectable once that work has finished."""
        if e.ref_count <= 0:
            raise StoreError("unbalanced unpin")
        e.epoch = max(e.epoch, self.record_epoch(stream))
        e.ref_count -= 1
        if e.ref_count == 0 and self.entries.get(e.id) is e:
            self._queue(e)

    def garbage_collect(self, target_bytes: int | None = None) -> int:
        """Evict unpinned entries LRU-first until `target_bytes` (default gc_target_fraction x
        capacity) are freed, stopping at the first entry whose epoch is still running."""
        done = self.poll_epochs()
        if target_bytes is None:
            target_bytes = int(self.gc_target_fraction * self.capacity)
        freed = 0
        while freed < target_bytes and self._lru:
            stamp, _, id = self._lru[0]
            e = self.entries.get(id)
            if e is None or e.ref_count > 0 or e.lru_stamp != stamp:
                heapq.heappop(self._lru)  # superseded queue item
                continue
            if e.epoch > done:
                break
            heapq.heappop(self._lru)
            self._remove(e, reuse=True, epoch=e.epoch)
            self.evictions += 1
            freed += e.size_q
        if freed < target_bytes:
            self.flush_buckets()
        return freed

    def make_room(self, nbytes: int) -> Allocation:
        """allocate(), collecting garbage (and, when only running epochs stand in the way, waiting
        for the oldest of them) until the request fits; raises when pinned entries fill the store."""
        while True:
            try:
                return self.allocate(nbytes)
            except ReclamationNeeded:
                pass
            want = max(quantize_size(int(nbytes), self.mantissa_bits), int(self.gc_target_fraction * self.capacity))
            if self.garbage_collect(want) > 0:
                continue
            self.flush_buckets()
            try:
                return self.allocate(nbytes)
            except ReclamationNeeded:
                pass
            if not self._pending:
                raise ReclamationNeeded(f"device store pinned full ({self.occupancy()}/{self.capacity})")
            self.wait_epoch(self._pending[0][0])

    # -- typed conveniences ---------------------------------------------------------------

    def put(self, id, tensor: torch.Tensor, state: ChunkState = ChunkState.FINAL) -> Entry:
        """Copy a device tensor into the store (collecting garbage if the budget is full)."""
        t = tensor.contiguous()
        nbytes = t.numel() * t.element_size()
        alloc = self.make_room(nbytes)
        alloc.buffer[:nbytes].copy_(t.view(-1).view(torch.uint8), non_blocking=True)
        return self.insert(id, alloc, nbytes, state)

    def get(self, id, dtype, shape, min_state: ChunkState = ChunkState.FINAL):
        """(pinned entry, typed view of its payload) or None; unpin (or retire) the entry when done."""
        e = self.lookup(id, min_state)
        if e is None:
            return None
        return e, e.payload.view(dtype).view(shape)

    def reserve(self, id, nbytes: int) -> Entry:
        """A pinned IN_FLIGHT entry of `nbytes` to be written by queued work; `publish` it."""
        if id in self.entries:
            raise StoreError(f"{id!r} is already in the store")
        alloc = self.make_room(nbytes)
        e = self.insert(id, alloc, nbytes, ChunkState.IN_FLIGHT, epoch=self.current_epoch)
        e.ref_count += 1
        return e

    def publish(self, e: Entry, state: ChunkState = ChunkState.FINAL, stream=None) -> None:
        """Mark a reserved entry complete once the work queued on `stream` so far has run."""
        e.state = ChunkState(state)
        self.retire(e, stream)
