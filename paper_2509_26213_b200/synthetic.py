"""Deterministic synthetic inputs for the random-walker configs.

Two-blob phantom on normalised coordinates u = g / (n - 1):
background 0.1; blob A = ball at (0.3, 0.5, 0.5), radius 0.20, +0.7;
blob B = ball at (0.7, 0.5, 0.5), radius 0.15, +0.5; plus N(0, 0.05^2) noise
drawn in float64 from ``np.random.default_rng(0xC0FFEE)`` (the reference
test fixture seed, `pkg/tests/conftest.py:8-10`) and cast to float32.
2D images use the first two coordinates.  Time series shift both blob
centres along axis 1 by 0.1 * t / (T - 1).

Seed sets (U8; 0 unseeded, 1 foreground, 2 background):
S1 = foreground ball r = 0.04 at blob A's centre, background = the slabs
u0 <= 0.03 and u1 <= 0.03;  S2 = the same with the ball at blob B's centre.

`phantom_device` / `seeds_device` build the same geometry with torch on the
GPU for sizes where host generation is impractical (1024^3); their noise
comes from torch's generator, so they are bit-compatible with the numpy
version only in the noiseless part.
"""

from __future__ import annotations

import numpy as np

RNG_SEED = 0xC0FFEE
BACKGROUND = 0.1
BLOB_A = ((0.3, 0.5, 0.5), 0.20, 0.7)
BLOB_B = ((0.7, 0.5, 0.5), 0.15, 0.5)
NOISE_SIGMA = 0.05
SEED_RADIUS = 0.04
BG_SLAB = 0.03


def _coords(shape):
    axes = []
    for i, n in enumerate(shape):
        u = np.arange(n, dtype=np.float64) / max(n - 1, 1)
        axes.append(u.reshape([-1 if j == i else 1 for j in range(len(shape))]))
    return axes


def _blob_centres(t=0, steps=1):
    shift = 0.1 * t / (steps - 1) if steps > 1 else 0.0
    out = []
    for centre, radius, value in (BLOB_A, BLOB_B):
        c = list(centre)
        c[1] += shift
        out.append((tuple(c), radius, value))
    return out


def phantom(shape, seed: int = RNG_SEED, noise: float = NOISE_SIGMA, t: int = 0,
            steps: int = 1) -> np.ndarray:
    shape = tuple(int(s) for s in shape)
    u = _coords(shape)
    vol = np.full(shape, BACKGROUND, dtype=np.float64)
    for centre, radius, value in _blob_centres(t, steps):
        d2 = sum((u[i] - centre[i]) ** 2 for i in range(len(shape)))
        vol = vol + value * (d2 <= radius * radius)
    if noise:
        vol = vol + np.random.default_rng(seed).normal(0.0, noise, size=shape)
    return vol.astype(np.float32)


def _blob_boxes(shape, t, steps):
    """Per blob: (f64 value added inside it, per-dim index range of its bounding box)."""
    u = _coords(shape)
    out = []
    for centre, radius, value in _blob_centres(t, steps):
        box = []
        for i, n in enumerate(shape):
            inside = np.nonzero(np.abs(u[i].ravel() - centre[i]) <= radius + 1e-12)[0]
            box.append((int(inside[0]), int(inside[-1]) + 1) if len(inside) else (0, 0))
        out.append((centre, radius, value, box))
    return u, out


def phantom_streamed(shape, seed: int = RNG_SEED, noise: float = NOISE_SIGMA, t: int = 0, steps: int = 1,
                     slab: int = 32, out: np.ndarray | None = None) -> np.ndarray:
    """`phantom` generated `slab` planes (dim 0) at a time, bit-identical to `phantom(shape, ...)`:
    the same normal stream (drawn slab by slab from one generator) and, per element, the same
    float64 value f32((BACKGROUND + v_A m_A + v_B m_B) + noise) — the blob term is evaluated only
    inside each blob's bounding box (outside it the masks are 0 and the sum is BACKGROUND exactly;
    the blobs are disjoint).  Temporaries stay slab-sized: 1024^3 needs the 4 GiB f32 result only.
    `out`: an f32 array (e.g. pinned host memory viewed through numpy) to fill."""
    shape = tuple(int(s) for s in shape)
    u, blobs = _blob_boxes(shape, t, steps)
    rng = np.random.default_rng(seed) if noise else None
    if out is None:
        out = np.empty(shape, dtype=np.float32)
    nd = len(shape)
    for z0 in range(0, shape[0], slab):
        z1 = min(z0 + slab, shape[0])
        sub = (z1 - z0,) + shape[1:]
        base = np.full(sub, BACKGROUND, dtype=np.float64)
        for centre, radius, value, box in blobs:
            lo = [max(box[0][0], z0)] + [b[0] for b in box[1:]]
            hi = [min(box[0][1], z1)] + [b[1] for b in box[1:]]
            if any(h <= l for l, h in zip(lo, hi)):
                continue
            us = [u[i].reshape(-1)[lo[i]:hi[i]].reshape([-1 if j == i else 1 for j in range(nd)]) for i in range(nd)]
            d2 = sum((us[i] - centre[i]) ** 2 for i in range(nd))
            sel = (slice(lo[0] - z0, hi[0] - z0),) + tuple(slice(l, h) for l, h in zip(lo[1:], hi[1:]))
            base[sel] = base[sel] + value * (d2 <= radius * radius)
        if noise:
            base += rng.normal(0.0, noise, size=sub)
        out[z0:z1] = base
    return out


def seeds_streamed(shape, which: str = "S1", t: int = 0, steps: int = 1, slab: int = 64,
                   out: np.ndarray | None = None) -> np.ndarray:
    """`seeds` generated slab by slab (bit-identical; bounded temporaries)."""
    shape = tuple(int(s) for s in shape)
    if out is None:
        out = np.empty(shape, dtype=np.uint8)
    u = _coords(shape)
    (ca, _, _), (cb, _, _) = _blob_centres(t, steps)
    centre = {"S1": ca, "S2": cb}[which]
    for z0 in range(0, shape[0], slab):
        z1 = min(z0 + slab, shape[0])
        sub = (z1 - z0,) + shape[1:]
        us = [u[0][z0:z1]] + u[1:]
        o = np.zeros(sub, dtype=np.uint8)
        bg = (us[0] <= BG_SLAB) | (us[1] <= BG_SLAB)
        o[np.broadcast_to(bg, sub)] = 2
        d2 = sum((us[i] - centre[i]) ** 2 for i in range(len(shape)))
        o[np.broadcast_to(d2 <= SEED_RADIUS * SEED_RADIUS, sub)] = 1
        out[z0:z1] = o
    return out


def series_timestep(shape, t: int, steps: int, slab: int = 32, out: np.ndarray | None = None) -> np.ndarray:
    """Timestep t of the config-5 4-D series: the phantom with both blobs shifted along axis 1 by
    0.1 t / (T - 1) and its own noise draw (seed RNG_SEED + t)."""
    return phantom_streamed(shape, seed=RNG_SEED + t, t=t, steps=steps, slab=slab, out=out)


def seeds(shape, which: str = "S1", t: int = 0, steps: int = 1) -> np.ndarray:
    shape = tuple(int(s) for s in shape)
    u = _coords(shape)
    (ca, _, _), (cb, _, _) = _blob_centres(t, steps)
    centre = {"S1": ca, "S2": cb}[which]
    out = np.zeros(shape, dtype=np.uint8)
    bg = (u[0] <= BG_SLAB) | (u[1] <= BG_SLAB)
    out[np.broadcast_to(bg, shape)] = 2
    d2 = sum((u[i] - centre[i]) ** 2 for i in range(len(shape)))
    out[np.broadcast_to(d2 <= SEED_RADIUS * SEED_RADIUS, shape)] = 1
    return out


# ---------------------------------------------------------------------------
# device-side generation (bench-scale volumes)


def _coords_t(shape, device):
    import torch

    axes = []
    for i, n in enumerate(shape):
        u = torch.arange(n, dtype=torch.float32, device=device) / max(n - 1, 1)
        axes.append(u.reshape([-1 if j == i else 1 for j in range(len(shape))]))
    return axes


def phantom_device(shape, device="cuda", seed: int = RNG_SEED, noise: float = NOISE_SIGMA,
                   t: int = 0, steps: int = 1):
    import torch

    shape = tuple(int(s) for s in shape)
    u = _coords_t(shape, device)
    vol = torch.full(shape, BACKGROUND, dtype=torch.float32, device=device)
    for centre, radius, value in _blob_centres(t, steps):
        d2 = sum((u[i] - centre[i]) ** 2 for i in range(len(shape)))
        vol += value * (d2 <= radius * radius).to(torch.float32)
    if noise:
        gen = torch.Generator(device=device)
        gen.manual_seed(seed + t)
        vol += noise * torch.randn(shape, generator=gen, device=device, dtype=torch.float32)
    return vol


def seeds_device(shape, which: str = "S1", device="cuda", t: int = 0, steps: int = 1):
    import torch

    shape = tuple(int(s) for s in shape)
    u = _coords_t(shape, device)
    (ca, _, _), (cb, _, _) = _blob_centres(t, steps)
    centre = {"S1": ca, "S2": cb}[which]
    out = torch.zeros(shape, dtype=torch.uint8, device=device)
    bg = (u[0] <= BG_SLAB) | (u[1] <= BG_SLAB)
    out.masked_fill_(bg.expand(shape), 2)
    d2 = sum((u[i] - centre[i]) ** 2 for i in range(len(shape)))
    out.masked_fill_((d2 <= SEED_RADIUS * SEED_RADIUS).expand(shape), 1)
    return out
