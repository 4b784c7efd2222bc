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
