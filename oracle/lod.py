"""Dense restatement of the reference LOD pyramid (test infrastructure only).

The reference builds level k+1 of a pyramid as
``downsample_mean(separable_conv(level_k, [[.25, .5, .25]] * d))``
(`pkg/src/chunkcast/ops.py:714-727`), chunk by chunk.  Each chunk kernel
works in float64 and casts back to the element type:

* `separable_conv` (`ops.py:471-530`): gather the chunk plus a radius-1 halo
  as float64 (`assemble_region`, `ops.py:443-464`), replicate edge elements
  outside the volume (`np.pad(mode="edge")`, `ops.py:509-515`), correlate
  dimension 0, then 1, ... with ``acc += k[j] * block[j:j+n]`` in tap order
  (`_conv1d`, `ops.py:533-548`), cast to float32 (`cast_array`, `ops.py:44-52`).
* `downsample_mean` (`ops.py:611-661`): pairwise ``(a + b) * 0.5`` along
  dimension 0, then 1, ...; an odd tail element is kept as is
  (`_pairwise_mean`, `ops.py:664-676`), then cast to float32.

The dense versions below perform the identical IEEE operations in the same
order on the same values, so they are bit-identical to the chunked
reference (checked against frozen reference outputs in `tests/golden/`).
"""

from __future__ import annotations

import numpy as np

SMOOTHING_KERNEL = (0.25, 0.5, 0.25)  # ops.py:679


def separable_conv_clamp(data: np.ndarray, kernels) -> np.ndarray:
    """Float64 per-dimension correlation with edge clamping (ops.py:471-548)."""
    out = np.asarray(data, dtype=np.float64)
    for dim, k in enumerate(kernels):
        k = [float(c) for c in k]
        r = len(k) // 2
        pad = [(r, r) if i == dim else (0, 0) for i in range(out.ndim)]
        block = np.pad(out, pad, mode="edge") if r else out
        n = out.shape[dim]
        acc = np.zeros(out.shape, dtype=np.float64)
        for j, c in enumerate(k):
            sel = [slice(None)] * out.ndim
            sel[dim] = slice(j, j + n)
            acc += c * block[tuple(sel)]
        out = acc
    return out


def pairwise_mean(data: np.ndarray, dims=None) -> np.ndarray:
    """Factor-2 mean; ragged tail keeps the lone element (ops.py:664-676)."""
    out = np.asarray(data, dtype=np.float64)
    dims = range(out.ndim) if dims is None else sorted(dims)
    for dim in dims:
        n = out.shape[dim]
        even = n - n % 2
        a = [slice(None)] * out.ndim
        b = [slice(None)] * out.ndim
        a[dim] = slice(0, even, 2)
        b[dim] = slice(1, even, 2)
        paired = (out[tuple(a)] + out[tuple(b)]) * 0.5
        if n % 2:
            t = [slice(None)] * out.ndim
            t[dim] = slice(n - 1, n)
            paired = np.concatenate([paired, out[tuple(t)]], axis=dim)
        out = paired
    return out


def lod_down(level: np.ndarray) -> np.ndarray:
    """One pyramid step: f32(mean(f32(conv(level)))) (ops.py:721-723)."""
    level = np.asarray(level, dtype=np.float32)
    conv = separable_conv_clamp(level, [SMOOTHING_KERNEL] * level.ndim).astype(np.float32)
    return pairwise_mean(conv).astype(np.float32)


def num_lod_levels(size, chunk) -> int:
    """Level count of `build_lod`: halve until every dim fits one chunk (ops.py:720)."""
    size = [int(s) for s in size]
    n = 1
    while any(s > c for s, c in zip(size, chunk)):
        size = [-(-s // 2) for s in size]
        n += 1
    return n


def lod_chain(volume: np.ndarray, chunk, levels: int | None = None) -> list:
    """Levels 0..L-1 of `build_lod(source_from_array(volume, chunk))`.

    `levels=None` takes every level the reference would build; a smaller
    value truncates the chain (the hierarchical random walker's level cap).
    """
    total = num_lod_levels(volume.shape, chunk)
    if levels is None:
        levels = total
    if not 1 <= levels <= total:
        raise ValueError(f"levels={levels} outside 1..{total} for size {volume.shape}, chunk {chunk}")
    out = [np.asarray(volume, dtype=np.float32)]
    for _ in range(levels - 1):
        out.append(lod_down(out[-1]))
    return out


def lod_down_slabbed(level: np.ndarray, slab: int = 32) -> np.ndarray:
    """`lod_down` computed `slab` coarse planes (dim 0) at a time — bit-identical, with float64
    temporaries bounded by the slab (1024^3 levels).

    Coarse planes [j0, j1) read fine planes [2 j0 - 1, 2 j1 + 1) through the radius-1 dim-0 taps.
    Each slab is convolved over that window: interior window edges only change the discarded
    outermost planes, and where the window meets the level's border the edge padding is the
    reference's own clamp (`ops.py:509-515`); the per-element float64 operations are unchanged.
    """
    level = np.asarray(level, dtype=np.float32)
    n = level.shape[0]
    m = -(-n // 2)
    out = np.empty((m,) + tuple(-(-s // 2) for s in level.shape[1:]), dtype=np.float32)
    for j0 in range(0, m, slab):
        j1 = min(j0 + slab, m)
        f0, f1 = max(2 * j0 - 1, 0), min(2 * j1 + 1, n)
        conv = separable_conv_clamp(level[f0:f1], [SMOOTHING_KERNEL] * level.ndim).astype(np.float32)
        keep = conv[2 * j0 - f0:min(2 * j1, n) - f0]
        out[j0:j1] = pairwise_mean(keep).astype(np.float32)
    return out
