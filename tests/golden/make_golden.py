"""Regenerate the frozen fixtures under tests/golden/ (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

* `lod_reference.npz` — pyramids computed by the REFERENCE itself:
  `chunkcast.ops.build_lod(source_from_array(x, chunk))` resolved through
  `chunkcast.Engine` (`pkg/src/chunkcast/ops.py:714-727`, `engine.py:423-448`).
  These pin `oracle.lod` (bit-exact) and the CUDA LOD kernel.
* `plct/` — chunked tensor files written by the reference's `tensorfile` module
  (`import_raw`, `_ChunkWriter`, `build_lod_offline`; `tensorfile.py:149-165, 108-146, 307-341`),
  with the arrays they hold (`*.npy`).
* `rw_*.npz` — random-walker outputs of the float64 oracle (`oracle.rw`,
  tol 1e-10) on the synthetic configs.  The reference has no random walker,
  so these are oracle outputs, not reference outputs (parity unpinned).

`/root/reference` is not available on the GPU box; only the frozen files
travel.  `MANIFEST.json` holds SHA-256 digests of inputs and outputs.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import rw  # noqa: E402
from paper_2509_26213_b200 import synthetic as syn  # noqa: E402

LOD_CASES = {
    # name: (shape, chunk, dtype seed)
    "r3d": ((21, 18, 13), (8, 8, 8)),
    "r2d": ((37, 29), (8, 8)),
    "r1d": ((11,), (3,)),
    "phantom3d": ((64, 64, 64), (16, 16, 16)),
    "phantom2d": ((96, 80), (16, 16)),
}

RW_CASES = {
    # name: (shape, seedset, brick, levels)
    "c1_s1": ((64, 64, 64), "S1", (32, 32, 32), 1),
    "c1_s2": ((64, 64, 64), "S2", (32, 32, 32), 1),
    "h3d_s1": ((48, 48, 48), "S1", (16, 16, 16), 2),
    "h3d_ragged_s2": ((40, 36, 28), "S2", (16, 16, 16), 2),
    "h2d_s1": ((128, 128), "S1", (32, 32), 3),
    "h2d_s2": ((96, 112), "S2", (32, 32), 2),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def lod_input(name, shape):
    if name.startswith("phantom"):
        return syn.phantom(shape)
    rng = np.random.default_rng(0xC0FFEE + len(shape))
    return rng.random(shape, dtype=np.float32)


def make_lod(manifest):
    from chunkcast import ops
    from chunkcast.engine import Engine, EngineConfig
    from chunkcast.store import StoreConfig

    arrays = {}
    with Engine(EngineConfig(stores=StoreConfig(ram_capacity=1 << 28))) as eng:
        for name, (shape, chunk) in LOD_CASES.items():
            x = lod_input(name, shape)
            pyr = ops.build_lod(ops.source_from_array(x, chunk))
            if not name.startswith("phantom"):  # phantoms are regenerated from synthetic.py
                arrays[f"{name}/input"] = x
            levels_sha = [sha(x)]
            for k in range(1, pyr.num_levels):
                node = pyr.node(k)
                chunks = eng.resolve(node)
                full = np.zeros(node.md.size, dtype=np.float32)
                for pos, arr in zip(node.md.chunk_positions(), chunks):
                    begin, end = node.md.chunk_logical_region(pos)
                    dst = tuple(slice(b, e) for b, e in zip(begin, end))
                    full[dst] = arr[tuple(slice(0, e - b) for b, e in zip(begin, end))]
                arrays[f"{name}/level{k}"] = full
                levels_sha.append(sha(full))
            manifest["lod"][name] = {
                "shape": list(shape), "chunk": list(chunk), "levels": pyr.num_levels,
                "input_sha256": sha(x),
                "levels_sha256": levels_sha,
            }
    np.savez_compressed(os.path.join(HERE, "lod_reference.npz"), **arrays)


def make_rw(manifest):
    params = rw.RWParams(beta=100.0, min_weight=1e-6, tol=1e-10, max_iter=20000)
    for name, (shape, which, brick, levels) in RW_CASES.items():
        vol = syn.phantom(shape)
        seeds = syn.seeds(shape, which)
        res = rw.hierarchical_random_walker(vol, seeds, brick, levels, params)
        out = {"labels": res.labels}
        for k, p in enumerate(res.prob):
            out[f"prob{k}"] = p.astype(np.float32)
        np.savez_compressed(os.path.join(HERE, f"rw_{name}.npz"), **out)
        manifest["rw"][name] = {
            "shape": list(shape), "seeds": which, "brick": list(brick), "levels": levels,
            "beta": params.beta, "min_weight": params.min_weight, "tol": params.tol,
            "input_sha256": sha(vol), "seeds_sha256": sha(seeds),
            "prob0_sha256": sha(out["prob0"]), "labels_sha256": sha(res.labels),
            "iterations_max": [int(i.max()) if len(i) else 0 for i in res.iterations],
        }
        print(name, manifest["rw"][name]["iterations_max"], flush=True)


C2_SUB = 4  # config-2 fixture: every 4th voxel per axis of the level-0 probabilities


def make_c2(manifest):
    """Config 2 at full size (256^3, 2 levels, 32^3 bricks, seeds S1), oracle at tol 1e-9 on 8
    threads (~3 min); the fixture keeps a strided subsample (64^3 points, ~1 MB)."""
    params = rw.RWParams(beta=100.0, min_weight=1e-6, tol=1e-9, max_iter=50000)
    shape = (256, 256, 256)
    vol = syn.phantom(shape)
    seeds = syn.seeds(shape, "S1")
    res = rw.hierarchical_random_walker(vol, seeds, (32, 32, 32), 2, params, threads=8)
    sub = tuple(slice(None, None, C2_SUB) for _ in shape)
    p = res.prob[0][sub].astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "rw_c2_sub4.npz"), prob0=p)
    manifest["rw_c2_sub4"] = {"shape": list(shape), "seeds": "S1", "brick": [32, 32, 32], "levels": 2,
                              "tol": params.tol, "stride": C2_SUB, "input_sha256": sha(vol),
                              "seeds_sha256": sha(seeds), "prob0_sub_sha256": sha(p)}


def make_c3like(manifest):
    """Config-3 structure at 2048^2 (64^2 tiles, all 6 levels down to a 64^2 whole level), oracle
    at tol 1e-9; the fixture keeps every 4th pixel per axis of level 0 (512^2 points)."""
    params = rw.RWParams(beta=100.0, min_weight=1e-6, tol=1e-9, max_iter=50000)
    shape = (2048, 2048)
    vol = syn.phantom(shape)
    seeds = syn.seeds(shape, "S1")
    res = rw.hierarchical_random_walker(vol, seeds, (64, 64), 6, params, threads=8)
    p = res.prob[0][::4, ::4].astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "rw_c3like_sub4.npz"), prob0=p)
    manifest["rw_c3like_sub4"] = {"shape": list(shape), "seeds": "S1", "brick": [64, 64], "levels": 6,
                                  "tol": params.tol, "stride": 4, "input_sha256": sha(vol),
                                  "seeds_sha256": sha(seeds), "prob0_sub_sha256": sha(p)}


PLCT_DIR = os.path.join(HERE, "plct")


def make_plct(manifest):
    """Chunked tensor files written by the REFERENCE (`chunkcast.tensorfile`): `import_raw` of
    f32 / u8 / u16x2 tensors, a hand-ordered file with absent chunks (`_ChunkWriter`), and the
    pyramids `build_lod_offline` materialises (smooth and plain).  They pin `plct.py` (reader,
    byte-identical writer) and the GPU `build_lod_offline` (byte-identical level files)."""
    from chunkcast import tensorfile as tf
    from chunkcast.engine import Engine, EngineConfig
    from chunkcast.model import ElementType, EmbeddingData, Scalar, TensorMetaData
    from chunkcast.store import StoreConfig

    os.makedirs(PLCT_DIR, exist_ok=True)
    for name in os.listdir(PLCT_DIR):
        os.remove(os.path.join(PLCT_DIR, name))
    rng = np.random.default_rng(0x9C7)
    cases = {
        "vol3d": (rng.random((40, 36, 28), dtype=np.float32), (16, 16, 16), Scalar.F32, 1, (0.5, 0.75, 1.0)),
        "seeds3d": (rng.integers(0, 3, (40, 36, 28)).astype(np.uint8), (16, 16, 16), Scalar.U8, 1, (0.5, 0.75, 1.0)),
        "img2d": (rng.random((37, 29), dtype=np.float32), (8, 8), Scalar.F32, 1, (1.0, 1.0)),
        "vec2d_u16x2": (rng.integers(0, 65535, (9, 7, 2)).astype(np.uint16), (4, 4), Scalar.U16, 2, (1.0, 2.0)),
    }
    entry = {}
    for name, (arr, chunk, scalar, lanes, spacing) in cases.items():
        raw = os.path.join(PLCT_DIR, f"{name}.raw")
        arr.tofile(raw)
        size = arr.shape[:-1] if lanes > 1 else arr.shape
        md = TensorMetaData(size, chunk, ElementType(scalar, lanes))
        out = os.path.join(PLCT_DIR, f"{name}.plct")
        tf.import_raw(raw, out, md, EmbeddingData(spacing))
        os.remove(raw)
        np.save(os.path.join(PLCT_DIR, f"{name}.npy"), arr)
        entry[name] = {"shape": list(arr.shape), "chunk": list(chunk), "lanes": lanes,
                       "spacing": list(spacing), "sha256": sha(arr)}
    # absent chunks and reverse file order, through the reference's writer
    arr = cases["img2d"][0]
    md = TensorMetaData(arr.shape, (8, 8), ElementType(Scalar.F32, 1))
    positions = list(md.chunk_positions())
    with tf._ChunkWriter(os.path.join(PLCT_DIR, "sparse2d.plct"), md, (1.0, 1.0)) as w:
        for k, pos in enumerate(reversed(positions)):
            if k % 3 == 1:
                continue  # absent: reads as zeros
            begin, end = md.chunk_logical_region(pos)
            buf = np.zeros((8, 8), np.float32)
            buf[tuple(slice(0, e - b) for b, e in zip(begin, end))] = arr[tuple(slice(b, e) for b, e in zip(begin, end))]
            w.write_chunk(pos, buf)
    # a volume with uniform chunks (and one NaN) for the constant-chunk tables
    blocky = np.zeros((40, 36, 28), np.float32)
    blocky[16:, :, :] = 0.25
    blocky[16:32, 16:32, 16:] = rng.random((16, 16, 12), dtype=np.float32)
    blocky[5, 5, 5] = np.nan
    raw = os.path.join(PLCT_DIR, "blocky3d.raw")
    blocky.tofile(raw)
    tf.import_raw(raw, os.path.join(PLCT_DIR, "blocky3d.plct"),
                  TensorMetaData(blocky.shape, (16, 16, 16), ElementType(Scalar.F32, 1)), EmbeddingData((1.0, 1.0, 1.0)))
    os.remove(raw)
    np.save(os.path.join(PLCT_DIR, "blocky3d.npy"), blocky)
    from chunkcast import ops as rops
    with Engine(EngineConfig(stores=StoreConfig(ram_capacity=1 << 28))) as eng:
        tf.save_tensor(rops.build_const_chunk_table(tf.open_chunked(os.path.join(PLCT_DIR, "seeds3d.plct"))),
                       os.path.join(PLCT_DIR, "seeds3d.ctab.plct"), eng)
        tf.build_lod_offline(os.path.join(PLCT_DIR, "blocky3d.plct"), os.path.join(PLCT_DIR, "blocky3d_ct.json"), eng,
                             const_tables=True)
        tf.build_lod_offline(os.path.join(PLCT_DIR, "vol3d.plct"), os.path.join(PLCT_DIR, "vol3d_pyr.json"), eng)
        tf.build_lod_offline(os.path.join(PLCT_DIR, "img2d.plct"), os.path.join(PLCT_DIR, "img2d_plain.json"), eng,
                             smooth=False)
    manifest["plct"] = {"cases": entry, "files": {n: hashlib.sha256(open(os.path.join(PLCT_DIR, n), "rb").read())
                                                  .hexdigest() for n in sorted(os.listdir(PLCT_DIR))}}


def main():
    manifest = {"lod": {}, "rw": {}}
    if "--plct-only" in sys.argv:
        path = os.path.join(HERE, "MANIFEST.json")
        with open(path) as f:
            manifest = json.load(f)
        make_plct(manifest)
        with open(path, "w") as f:
            json.dump(manifest, f, indent=1, sort_keys=True)
        return
    path = os.path.join(HERE, "MANIFEST.json")
    if "--c2-only" in sys.argv or "--c3like-only" in sys.argv:  # heavy fixtures, merged into the manifest
        with open(path) as f:
            manifest = json.load(f)
        if "--c2-only" in sys.argv:
            make_c2(manifest)
        if "--c3like-only" in sys.argv:
            make_c3like(manifest)
    else:
        make_lod(manifest)
        make_rw(manifest)
        make_plct(manifest)
        if "--c2" in sys.argv:
            make_c2(manifest)
    with open(path, "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
