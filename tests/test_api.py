"""Public entry points (`api.segment`, `api.segment_many`) on host buffers.

`segment_many` overlaps uploads / downloads with the neighbouring volumes'
compute on separate streams; its results must be byte-identical to one
`segment` call per volume (same kernels, same workspace decisions).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2509_26213_b200 import api, synthetic  # noqa: E402
from paper_2509_26213_b200.config import RWConfig  # noqa: E402


def _case(shape, kind):
    return (torch.from_numpy(synthetic.phantom(shape)).pin_memory(),
            torch.from_numpy(synthetic.seeds(shape, kind)).pin_memory())


def test_segment_host_roundtrip_matches_device():
    vol, sd = _case((64, 64, 64), "S1")
    cfg = RWConfig(tol=1e-6)
    p_h, l_h = api.segment(vol, sd, (32, 32, 32), 2, cfg)
    p_d, l_d = api.segment(vol.cuda(), sd.cuda(), (32, 32, 32), 2, cfg)
    torch.cuda.synchronize()
    assert not p_h.is_cuda and p_d.is_cuda
    np.testing.assert_array_equal(p_h.numpy(), p_d.cpu().numpy())
    np.testing.assert_array_equal(l_h.numpy(), l_d.cpu().numpy())


@pytest.mark.parametrize("n_out", [2, 4])
def test_segment_many_matches_single_calls(n_out):
    shape = (64, 64, 96)
    inputs = [_case(shape, k) for k in ("S1", "S2", "S1", "S2")]
    inputs[2] = (inputs[2][0] * 0.5, inputs[2][1])  # a different volume
    cfg = RWConfig(tol=1e-6)
    outs = [(torch.empty(shape, dtype=torch.float32, pin_memory=True),
             torch.empty(shape, dtype=torch.uint8, pin_memory=True)) for _ in range(n_out)]
    ref = [tuple(t.clone() for t in api.segment(v, s, (32, 32, 32), 2, cfg)) for v, s in inputs]
    if n_out < len(inputs):  # cyclic outputs: check each result as it would be read, one call per volume
        for k, (v, s) in enumerate(inputs):
            got = api.segment_many([(v, s)], (32, 32, 32), 2, cfg, outputs=outs)
            np.testing.assert_array_equal(got[0][0].numpy(), ref[k][0].numpy())
        with pytest.raises(ValueError):  # fewer outputs than inputs needs the explicit opt-in
            api.segment_many(inputs, (32, 32, 32), 2, cfg, outputs=outs)
        got = api.segment_many(inputs, (32, 32, 32), 2, cfg, outputs=outs, cyclic_outputs=True)
        last = (len(inputs) - 1) % n_out
        np.testing.assert_array_equal(outs[last][0].numpy(), ref[-1][0].numpy())
        np.testing.assert_array_equal(outs[last][1].numpy(), ref[-1][1].numpy())
    else:
        got = api.segment_many(inputs, (32, 32, 32), 2, cfg, outputs=outs)
        for (p, l), (rp, rl) in zip(got, ref):
            np.testing.assert_array_equal(p.numpy(), rp.numpy())
            np.testing.assert_array_equal(l.numpy(), rl.numpy())


@pytest.mark.parametrize("shape,brick,levels", [((96, 64, 64), (32, 32, 32), 2), ((256, 192), (64, 64), 2),
                                                ((70, 40, 48), (16, 16, 16), 2)])
def test_level0_chunks_bytes_identical(shape, brick, levels):
    """Level 0 solved in slabs of brick rows (api.segment_many's download overlap) = one solve."""
    from paper_2509_26213_b200 import device

    vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
    sd = torch.from_numpy(synthetic.seeds(shape, "S1")).cuda()
    cfg = RWConfig(tol=1e-6)
    a = device.hierarchical_random_walker(vol, sd, brick, levels, cfg)
    seen = []
    b = device.hierarchical_random_walker(vol, sd, brick, levels, cfg, level0_chunks=3,
                                          on_level0_chunk=lambda r0, r1, p, l: seen.append((r0, r1)))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(a.prob.cpu().numpy(), b.prob.cpu().numpy())
    np.testing.assert_array_equal(a.labels.cpu().numpy(), b.labels.cpu().numpy())
    assert seen[0][0] == 0 and seen[-1][1] == shape[0] and all(x[1] == y[0] for x, y in zip(seen, seen[1:]))
    for key in ("bricks", "iterations_sum", "unknowns", "unknown_iterations", "iterations_max"):
        assert a.stats[0][key] == b.stats[0][key]


def test_segment_series_matches_per_timestep_calls():
    t_steps, shape = 3, (64, 64, 64)
    vol = torch.stack([torch.from_numpy(synthetic.phantom(shape, t=t, steps=t_steps)) for t in range(t_steps)])
    sd = torch.stack([torch.from_numpy(synthetic.seeds(shape, "S1", t=t, steps=t_steps)) for t in range(t_steps)])
    vol, sd = vol.pin_memory(), sd.pin_memory()
    cfg = RWConfig(tol=1e-6)
    prob, labels = api.segment_series(vol, sd, (32, 32, 32), 2, cfg)
    for t in range(t_steps):
        p, l = api.segment(vol[t].clone(), sd[t].clone(), (32, 32, 32), 2, cfg)
        np.testing.assert_array_equal(prob[t].numpy(), p.numpy())
        np.testing.assert_array_equal(labels[t].numpy(), l.numpy())
    assert not np.array_equal(prob[0].numpy(), prob[-1].numpy())  # the blobs move


def test_segment_many_default_outputs_are_distinct():
    """Without `outputs`, every volume gets its own result buffers (no cyclic aliasing)."""
    shape = (64, 64, 64)
    inputs = [_case(shape, k) for k in ("S1", "S2", "S1")]
    inputs[2] = (inputs[2][0] * 0.5, inputs[2][1])
    cfg = RWConfig(tol=1e-6)
    got = api.segment_many(inputs, (32, 32, 32), 2, cfg)
    assert len({p.data_ptr() for p, _ in got}) == 3
    for (p, l), (v, s) in zip(got, inputs):
        rp, rl = api.segment(v, s, (32, 32, 32), 2, cfg)
        np.testing.assert_array_equal(p.numpy(), rp.numpy())
        np.testing.assert_array_equal(l.numpy(), rl.numpy())


@pytest.mark.parametrize("shape,brick,levels", [((64, 64, 64), (64, 64, 64), 1), ((64, 64, 64), (32, 32, 32), 1),
                                                ((96, 80), (96, 80), 1)])
def test_single_level_host_path(shape, brick, levels):
    """A one-level hierarchy through the host API downloads its (whole-level) result."""
    vol, sd = _case(shape, "S1")
    cfg = RWConfig(tol=1e-6)
    out_p = torch.full(shape, float("nan"), dtype=torch.float32).pin_memory()
    out_l = torch.full(shape, 7, dtype=torch.uint8).pin_memory()
    p_h, l_h = api.segment(vol, sd, brick, levels, cfg, out_prob=out_p, out_labels=out_l)
    p_d, l_d = api.segment(vol.cuda(), sd.cuda(), brick, levels, cfg)
    torch.cuda.synchronize()
    assert not np.isnan(p_h.numpy()).any()
    np.testing.assert_array_equal(p_h.numpy(), p_d.cpu().numpy())
    np.testing.assert_array_equal(l_h.numpy(), l_d.cpu().numpy())


@pytest.mark.gpu
@pytest.mark.parametrize("shape,brick,levels,roi", [
    ((128, 96, 64), (32, 32, 32), 3, ((40, 10, 5), (75, 50, 30))),
    ((128, 96, 64), (32, 32, 32), 3, ((0, 0, 0), (1, 1, 1))),
    ((96, 80, 72), (16, 16, 16), 3, ((30, 17, 40), (64, 80, 72))),   # streaming solver, ragged
    ((448, 320), (64, 64), 3, ((100, 200), (260, 320))),             # 2-D tile engine
])
def test_region_limited_solve_equals_full_solve(shape, brick, levels, roi):
    """The lazy, region-limited hierarchy (the reference's pull of only the needed chunks): the
    region's probabilities and labels are the full solve's, bit for bit, with far fewer bricks."""
    import torch

    from paper_2509_26213_b200 import device
    from paper_2509_26213_b200.config import RWConfig

    vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
    sd = torch.from_numpy(synthetic.seeds(shape, "S1")).cuda()
    full = device.hierarchical_random_walker(vol, sd, brick, levels, RWConfig())
    part = device.hierarchical_random_walker(vol, sd, brick, levels, RWConfig(), roi=roi)
    box = tuple(slice(a, b) for a, b in zip(*roi))
    assert torch.equal(part.prob[box], full.prob[box]) and torch.equal(part.labels[box], full.labels[box])
    assert part.stats[0]["bricks"] < full.stats[0]["bricks"]
    assert torch.isnan(part.prob).any() or part.stats[0]["bricks"] == full.stats[0]["bricks"]
    p, lab = api.segment(vol.cpu().numpy(), sd.cpu().numpy(), brick, levels, RWConfig(), roi=roi)
    assert torch.equal(p, full.prob[box].cpu()) and torch.equal(lab, full.labels[box].cpu())
