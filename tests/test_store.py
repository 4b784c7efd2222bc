"""HBM chunk store: the reference store's semantics (`store.py:73-83,
145-342`) on device buffers, with CUDA-event epochs, and the pyramid cache built on it."""

import pytest

from paper_2509_26213_b200.store import ChunkState, quantize_size


def test_quantize_size_matches_reference_rule():
    # granularity 2^max(0, floor(log2 s) - 8): at most 1/256 overshoot
    assert quantize_size(1) == 1 and quantize_size(255) == 255 and quantize_size(256) == 256
    assert quantize_size(511) == 511 and quantize_size(513) == 514 and quantize_size(1025) == 1028
    for s in (3, 1000, 4097, 10 ** 6, 123456789):
        q = quantize_size(s)
        g = 1 << max(0, s.bit_length() - 1 - 8)
        assert q >= s and q % g == 0 and q - s < g
    with pytest.raises(ValueError):
        quantize_size(0)


@pytest.mark.gpu
def test_buckets_budget_and_lru():
    import torch

    from paper_2509_26213_b200.store import AllocationTooLarge, DeviceStore, ReclamationNeeded

    st = DeviceStore(10_000, gc_target_fraction=0.5)
    a = st.allocate(1000)
    assert a.buffer.is_cuda and a.size_q == 1000 and st.occupancy() == 1000
    st.free_allocation(a)
    assert st.cached_bytes == 1000 and st.allocate(1000) is a  # bucket reuse
    st.free_allocation(a)
    with pytest.raises(AllocationTooLarge):
        st.allocate(20_000)
    for i in range(4):
        st.put(("x", i), torch.full((500,), float(i), device="cuda"))  # 2000 B each
    torch.cuda.synchronize()
    with pytest.raises(ReclamationNeeded):
        st.allocate(3000)  # 4 x 2000 live + 1000 cached + 3000 > 10000
    e, v = st.get(("x", 0), torch.float32, (500,))  # pins 0 and makes it most recent
    assert torch.equal(v, torch.zeros(500, device="cuda"))
    freed = st.garbage_collect()  # target 5000: evicts 1, 2, 3 (LRU order), never the pinned 0
    assert freed >= 4000 and ("x", 0) in st.entries and ("x", 1) not in st.entries
    st.unpin(e)
    assert st.get(("x", 3), torch.float32, (500,)) is None


@pytest.mark.gpu
def test_gc_stops_at_a_running_epoch():
    import torch

    from paper_2509_26213_b200.store import DeviceStore

    st = DeviceStore(1 << 30)
    s = torch.cuda.Stream()
    st.put("done", torch.ones(1024, device="cuda"))
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        torch.cuda._sleep(200_000_000)  # keep this stream busy
        st.put("busy", torch.ones(1024, device="cuda"))  # epoch recorded behind the sleep
    freed = st.garbage_collect(target_bytes=1 << 30)
    assert "done" not in st.entries and "busy" in st.entries  # stopped at the running epoch
    s.synchronize()
    st.garbage_collect(target_bytes=1 << 30)
    assert "busy" not in st.entries and freed > 0


@pytest.mark.gpu
def test_duplicate_insert_keeps_the_stronger_state():
    import torch

    from paper_2509_26213_b200.store import DeviceStore

    st = DeviceStore(1 << 20)
    st.put("k", torch.zeros(16, device="cuda"), ChunkState.PREVIEW)
    st.put("k", torch.ones(16, device="cuda"), ChunkState.FINAL)
    st.put("k", torch.full((16,), 2.0, device="cuda"), ChunkState.FINAL)  # equal state: first wins
    e, v = st.get("k", torch.float32, (16,))
    assert e.state == ChunkState.FINAL and torch.equal(v, torch.ones(16, device="cuda"))
    assert st.get("missing", torch.float32, (1,)) is None


@pytest.mark.gpu
def test_pyramid_store_reuses_levels():
    import torch

    from paper_2509_26213_b200 import _native, device, synthetic
    from paper_2509_26213_b200.config import RWConfig
    from paper_2509_26213_b200.store import DeviceStore

    shape, brick = (96, 64, 64), (32, 32, 32)
    vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
    seeds = torch.from_numpy(synthetic.seeds(shape, "S1")).cuda()
    ref = device.hierarchical_random_walker(vol, seeds, brick, 2, RWConfig())
    st = DeviceStore(1 << 28)
    a = device.hierarchical_random_walker(vol, seeds, brick, 2, RWConfig(), pyramid_store=st, pyramid_key="v")
    n0 = len(st.entries)
    b = device.hierarchical_random_walker(vol, seeds, brick, 2, RWConfig(), pyramid_store=st, pyramid_key="v")
    assert n0 == 1 and len(st.entries) == 1
    assert torch.equal(a.prob, ref.prob) and torch.equal(b.prob, ref.prob)


# -- shadow model: the reference Store and the arena store under the same operation sequence --


def _shadow_run(seed, sizes, capacity, n_ops=400, frac=0.25):
    import random

    from conftest import reference_package

    cc = reference_package()
    from chunkcast import store as rs

    from paper_2509_26213_b200 import store as ds

    rnd = random.Random(seed)
    ref = rs.StoreGroup(rs.StoreConfig(ram_capacity=capacity, gc_target_fraction=frac)).store(rs.RAM)
    ours = ds.DeviceStore(capacity, device="cpu", gc_target_fraction=frac)
    pins = []
    ids = [("c", i) for i in range(24)]
    steps = 0
    for _ in range(n_ops):
        op = rnd.random()
        if op < 0.5:
            id, size = rnd.choice(ids), rnd.choice(sizes)
            state = rnd.choice([rs.ChunkState.PREVIEW, rs.ChunkState.FINAL, rs.ChunkState.FINAL])
            got = []
            for st, mod in ((ref, rs), (ours, ds)):
                try:
                    got.append(st.allocate(size))
                except mod.ReclamationNeeded:
                    got.append(None)
            if (got[0] is None) != (got[1] is None):
                # only a fragmented arena may refuse what the accounting allows
                assert got[1] is None and ours.arena.largest_free() < ds._aligned(ds.quantize_size(size))
                return steps, ref, ours
            if got[0] is not None:
                ref.insert(id, got[0], size, rs.ChunkState(int(state)))
                ours.insert(id, got[1], size, ds.ChunkState(int(state)))
        elif op < 0.7:
            id = rnd.choice(ids)
            a, b = ref.lookup(id), ours.lookup(id)
            assert (a is None) == (b is None)
            if a is not None:
                pins.append((a.entry, b))
        elif op < 0.85 and pins:
            a, b = pins.pop(rnd.randrange(len(pins)))
            ref.unpin(a)
            ours.unpin(b)
        else:
            t = rnd.choice([None, rnd.choice(sizes), capacity])
            assert ref.garbage_collect(target_bytes=t) == ours.garbage_collect(target_bytes=t)
        steps += 1
        assert (ref.live_bytes, ref.cached_bytes) == (ours.live_bytes, ours.cached_bytes)
        assert {k: (e.state, e.size_bytes, e.ref_count) for k, e in ref.entries.items()} == \
               {k: (int(e.state), e.size_bytes, e.ref_count) for k, e in ours.entries.items()}
        assert ref.group.evictions == ours.evictions
        assert ours.occupancy() <= capacity and ours.arena.nbytes == capacity
    return steps, ref, ours


@pytest.mark.parametrize("seed", range(6))
def test_shadow_reference_store_one_bucket(seed):
    """One size: no fragmentation is possible, so every operation must agree with the reference
    `Store` (store.py:145-362) — accounting, entries, states, pins, evictions, GC results."""
    steps, _, ours = _shadow_run(seed, [4096], 16 * 4096)
    assert steps == 400 and ours.evictions > 0


@pytest.mark.parametrize("seed", range(8))
def test_shadow_reference_store_mixed_sizes(seed):
    """Mixed bucket sizes: agreement with the reference until (if ever) the arena is fragmented
    where the reference's unconstrained allocator is not."""
    steps, _, _ = _shadow_run(seed, [256, 768, 1024, 3000, 4096, 10_000], 48 * 1024)
    assert steps == 400  # (no fragmentation refusal occurs for these seeds)


def test_arena_extents_merge_and_never_overlap():
    import random

    from paper_2509_26213_b200.store import Arena

    rnd = random.Random(3)
    ar = Arena(1 << 16, "cpu")
    live = {}
    for _ in range(2000):
        if live and rnd.random() < 0.45:
            off = rnd.choice(list(live))
            ar.give(off, live.pop(off))
        else:
            n = 256 * rnd.randint(1, 16)
            off = ar.take(n)
            if off is not None:
                live[off] = n
        spans = sorted(live.items()) + list(zip(ar._starts, ar._lens))
        spans.sort()
        assert all(a + n <= b for (a, n), (b, _) in zip(spans, spans[1:]))  # disjoint
        assert sum(n for _, n in spans) == 1 << 16                          # and complete
        assert all(a + n < b for a, n, b in zip(ar._starts, ar._lens, ar._starts[1:]))  # free list merged
    for off, n in live.items():
        ar.give(off, n)
    assert ar._starts == [0] and ar._lens == [1 << 16]


@pytest.mark.gpu
def test_series_streams_through_a_budget_below_its_size():
    """Config-5 shape of use: a 4-D series segmented through a DeviceStore whose arena holds 3 of
    its 8 timesteps — same bytes as the private double-buffer path, the budget never exceeded,
    early timesteps evicted; with a budget holding the whole series a second pass uploads nothing."""
    import torch

    from paper_2509_26213_b200 import api, synthetic
    from paper_2509_26213_b200.config import RWConfig
    from paper_2509_26213_b200.store import DeviceStore

    T, shape = 8, (64, 64, 64)
    vol = torch.empty((T,) + shape, dtype=torch.float32, pin_memory=True)
    sd = torch.empty((T,) + shape, dtype=torch.uint8, pin_memory=True)
    for t in range(T):
        vol[t] = torch.from_numpy(synthetic.series_timestep(shape, t, T))
        sd[t] = torch.from_numpy(synthetic.seeds(shape, "S1", t=t, steps=T))
    cfg = RWConfig()
    ref_p, ref_l = api.segment_series(vol, sd, (32, 32, 32), 2, cfg)
    per = 5 * 64 ** 3
    st = DeviceStore(3 * per)
    p, l = api.segment_series(vol, sd, (32, 32, 32), 2, cfg, store=st)
    assert torch.equal(p, ref_p) and torch.equal(l, ref_l)
    assert st.peak_occupancy <= st.capacity and st.evictions >= T - 3 and st.misses == T
    big = DeviceStore(T * per + 4096)
    api.segment_series(vol, sd, (32, 32, 32), 2, cfg, store=big, series_id="s")
    p2, l2 = api.segment_series(vol, sd, (32, 32, 32), 2, cfg, store=big, series_id="s")
    assert big.hits == T and big.misses == T and big.evictions == 0
    assert torch.equal(p2, ref_p) and torch.equal(l2, ref_l)
