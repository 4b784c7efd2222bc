"""Chunked tensor files (PLCT) against files the reference wrote.

The fixtures under tests/golden/plct/ come from the reference's own `tensorfile` module
(`import_raw`, `_ChunkWriter`, `build_lod_offline`; tests/golden/make_golden.py --plct-only).
CPU tests: header parsing and packing, manifests, malformed files.  GPU tests: the streamed
reader and writer (`rwb_chunks_scatter` / `rwb_chunks_gather`) and the GPU `build_lod_offline`,
byte-identical to the reference's files.
"""

import filecmp
import json
import os
import shutil

import numpy as np
import pytest

from paper_2509_26213_b200 import plct

HERE = os.path.dirname(os.path.abspath(__file__))
G = os.path.join(HERE, "golden", "plct")
with open(os.path.join(HERE, "golden", "MANIFEST.json")) as _f:
    CASES = json.load(_f)["plct"]["cases"]


def gp(name):
    return os.path.join(G, name)


# ---------------------------------------------------------------------------- CPU


@pytest.mark.parametrize("name", sorted(CASES))
def test_header_of_reference_files(name):
    c = CASES[name]
    h = plct.read_header(gp(f"{name}.plct"))
    shape = tuple(c["shape"][:-1]) if c["lanes"] > 1 else tuple(c["shape"])
    assert h.size == shape and h.chunk == tuple(c["chunk"]) and h.lanes == c["lanes"]
    assert h.spacing == tuple(float(s) for s in c["spacing"])
    assert h.num_chunks == int(np.prod([-(-s // k) for s, k in zip(shape, c["chunk"])]))
    # import_raw writes every chunk, row-major, back to back
    assert np.array_equal(h.offsets, h.header_bytes + h.payload_bytes * np.arange(h.num_chunks, dtype=np.uint64))
    with open(gp(f"{name}.plct"), "rb") as f:
        head = f.read(h.header_bytes)
    assert plct._pack_header(h.size, h.chunk, h.code, h.lanes, h.spacing, h.offsets) == head
    assert os.path.getsize(gp(f"{name}.plct")) == h.header_bytes + h.num_chunks * h.payload_bytes


def test_sparse_file_header():
    h = plct.read_header(gp("sparse2d.plct"))
    n = h.num_chunks
    assert (h.offsets == 0).sum() == len([k for k in range(n) if k % 3 == 1])
    present = h.offsets[h.offsets != 0]
    assert np.all(np.diff(present.astype(np.int64)) < 0) or present.size <= 1  # written in reverse chunk order


@pytest.mark.parametrize("manifest", ["vol3d_pyr.json", "img2d_plain.json", "blocky3d_ct.json"])
def test_manifest_roundtrip(tmp_path, manifest):
    levels = plct.load_manifest(gp(manifest))
    assert all(os.path.exists(lv.path) for lv in levels)
    for lv in levels:
        for f in (lv.path, lv.const_table):
            if f:
                shutil.copy(f, tmp_path / os.path.basename(f))
    moved = [plct.PyramidLevel(str(tmp_path / os.path.basename(lv.path)), lv.spacing,
                               str(tmp_path / os.path.basename(lv.const_table)) if lv.const_table else None)
             for lv in levels]
    plct.save_manifest(moved, tmp_path / manifest)
    assert (tmp_path / manifest).read_text() == open(gp(manifest)).read()
    # spacing doubles per level (downsample_mean's embedding, ops.py:620-627)
    for a, b in zip(levels, levels[1:]):
        assert b.spacing == tuple(2 * s for s in a.spacing)


def test_malformed_files(tmp_path):
    good = open(gp("img2d.plct"), "rb").read()
    cases = {
        "magic": b"XLCT" + good[4:],
        "version": good[:4] + (2).to_bytes(4, "little") + good[8:],
        "code": good[:8] + bytes([9]) + good[9:],
        "truncated": good[:40],
        "offset": good[:-1],  # last payload runs past the end
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.plct"
        p.write_bytes(data)
        with pytest.raises(plct.PlctError):
            plct.read_header(p)
    bad = tmp_path / "m.json"
    bad.write_text('{"format": "other"}')
    with pytest.raises(plct.PlctError):
        plct.load_manifest(bad)


# ---------------------------------------------------------------------------- GPU


def _expected(name):
    return np.load(gp(f"{name}.npy"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("staging", [64 << 20, 3000])
def test_load_reference_files(name, staging):
    t, h = plct.load(gp(f"{name}.plct"), staging_bytes=staging)
    got = t.cpu().numpy()
    exp = _expected(name)
    assert got.dtype == exp.dtype and got.shape == exp.shape
    np.testing.assert_array_equal(got, exp)


@pytest.mark.gpu
def test_load_sparse_reverse_ordered_file():
    t, h = plct.load(gp("sparse2d.plct"), staging_bytes=1000)
    exp = _expected("img2d").copy()
    for idx in np.flatnonzero(h.offsets == 0):
        gy, gx = divmod(int(idx), h.grid[1])
        exp[gy * 8:(gy + 1) * 8, gx * 8:(gx + 1) * 8] = 0
    np.testing.assert_array_equal(t.cpu().numpy(), exp)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("staging", [64 << 20, 5000])
def test_save_is_byte_identical(tmp_path, name, staging):
    t, h = plct.load(gp(f"{name}.plct"))
    out = tmp_path / f"{name}.plct"
    plct.save(t, out, h.chunk, h.spacing, lanes=h.lanes, staging_bytes=staging)
    assert filecmp.cmp(out, gp(f"{name}.plct"), shallow=False)


@pytest.mark.gpu
@pytest.mark.parametrize("src,manifest,smooth", [("vol3d.plct", "vol3d_pyr.json", True),
                                                 ("img2d.plct", "img2d_plain.json", False)])
def test_build_lod_offline_matches_reference(tmp_path, src, manifest, smooth):
    shutil.copy(gp(src), tmp_path / src)
    levels = plct.build_lod_offline(tmp_path / src, tmp_path / manifest, smooth=smooth)
    ref = plct.load_manifest(gp(manifest))
    assert len(levels) == len(ref)
    for ours, theirs in zip(levels, ref):
        assert filecmp.cmp(ours.path, theirs.path, shallow=False), os.path.basename(theirs.path)
    assert (tmp_path / manifest).read_text() == open(gp(manifest)).read()


@pytest.mark.gpu
def test_const_chunk_table_matches_reference(tmp_path):
    t, h = plct.load(gp("seeds3d.plct"))
    table = plct.const_chunk_table(t, h.chunk)
    plct._save_const_table(t, h.chunk, tmp_path / "c.plct")
    assert filecmp.cmp(tmp_path / "c.plct", gp("seeds3d.ctab.plct"), shallow=False)
    ref, _ = plct.load(gp("seeds3d.ctab.plct"))
    assert torch_equal(table, ref)


def torch_equal(a, b):
    import torch
    return a.shape == b.shape and bool(torch.equal(a.view(torch.uint8), b.view(torch.uint8)))


@pytest.mark.gpu
def test_build_lod_offline_const_tables(tmp_path):
    shutil.copy(gp("blocky3d.plct"), tmp_path / "blocky3d.plct")
    levels = plct.build_lod_offline(tmp_path / "blocky3d.plct", tmp_path / "blocky3d_ct.json", const_tables=True)
    ref = plct.load_manifest(gp("blocky3d_ct.json"))
    assert len(levels) == len(ref)
    for ours, theirs in zip(levels, ref):
        assert filecmp.cmp(ours.path, theirs.path, shallow=False), os.path.basename(theirs.path)
        assert filecmp.cmp(ours.const_table, theirs.const_table, shallow=False), os.path.basename(theirs.const_table)
    assert (tmp_path / "blocky3d_ct.json").read_text() == open(gp("blocky3d_ct.json")).read()


@pytest.mark.gpu
def test_segment_file_equals_device_path(tmp_path):
    import torch

    from paper_2509_26213_b200 import device, synthetic
    from paper_2509_26213_b200.config import RWConfig

    shape, chunk = (64, 64, 64), (32, 32, 32)
    vol = torch.from_numpy(synthetic.phantom(shape)).cuda()
    seeds = torch.from_numpy(synthetic.seeds(shape, "S1")).cuda()
    plct.save(vol, tmp_path / "v.plct", chunk, (1.0, 1.0, 1.0))
    plct.save(seeds, tmp_path / "s.plct", chunk, (1.0, 1.0, 1.0))
    cfg = RWConfig(tol=1e-6)
    res = plct.segment_file(tmp_path / "v.plct", tmp_path / "s.plct", tmp_path / "p.plct", tmp_path / "l.plct",
                            levels=2, cfg=cfg)
    ref = device.hierarchical_random_walker(vol, seeds, chunk, 2, cfg)
    p, hp = plct.load(tmp_path / "p.plct")
    lab, hl = plct.load(tmp_path / "l.plct")
    assert hp.chunk == chunk and hl.code == 0
    assert torch.equal(p, ref.prob) and torch.equal(lab, ref.labels) and torch.equal(p, res.prob)
