"""oracle.rw pinned against an independent direct sparse solve, plus the
random-walker properties (Grady 2006) and reproduction of the frozen fixtures.

The reference has no random walker, so the RW oracle's parity is
unpinned against the reference; scipy's SuperLU on an explicitly assembled
per-brick Laplacian is the independent check of the restated maths, and the
whole hierarchy (seed projection, prolongation taps, per-brick Dirichlet
halos, level order) is checked against a chain composed from independently
restated pieces (test_hierarchy_matches_independent_composition).
"""

import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from conftest import GOLDEN, load_golden
from oracle import rw
from paper_2509_26213_b200 import synthetic as syn

with open(os.path.join(GOLDEN, "MANIFEST.json")) as f:
    MANIFEST = json.load(f)

TIGHT = rw.RWParams(tol=1e-12, max_iter=50_000)


def direct_brick_solve(vol, seeds, brick, bound, beta=100.0, wmin=1e-6):
    """Assemble each brick's Dirichlet problem explicitly and solve it with SuperLU."""
    vol = np.asarray(vol, np.float64)
    shape = vol.shape
    nd = len(shape)
    out = np.where(seeds == 1, 1.0, 0.0)
    if bound is not None:
        out = np.where(seeds == 0, bound, out)
    grid = [-(-s // b) for s, b in zip(shape, brick)]
    for h in np.ndindex(*grid):
        lo = [hi * b for hi, b in zip(h, brick)]
        hi_ = [min((x + 1) * b, s) for x, b, s in zip(h, brick, shape)]
        region = tuple(slice(a, b) for a, b in zip(lo, hi_))
        idx = {}
        for p in np.ndindex(*[b - a for a, b in zip(lo, hi_)]):
            g = tuple(a + q for a, q in zip(lo, p))
            if seeds[g] == 0:
                idx[g] = len(idx)
        if not idx:
            continue
        n = len(idx)
        rows, cols, vals = [], [], []
        rhs = np.zeros(n)
        for g, i in idx.items():
            diag = 0.0
            for k in range(nd):
                for s in (-1, 1):
                    nb = list(g)
                    nb[k] += s
                    nb = tuple(nb)
                    if not 0 <= nb[k] < shape[k]:
                        continue
                    w = max(np.exp(-beta * (vol[g] - vol[nb]) ** 2), wmin)
                    diag += w
                    if nb in idx:
                        rows.append(i)
                        cols.append(idx[nb])
                        vals.append(-w)
                    else:  # seed, or outside the brick
                        if seeds[nb] == 1:
                            v = 1.0
                        elif seeds[nb] == 2:
                            v = 0.0
                        else:
                            v = bound[nb]
                        rhs[i] += w * v
            rows.append(i)
            cols.append(i)
            vals.append(diag)
        A = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
        x = spla.spsolve(A.tocsc(), rhs)
        for g, i in idx.items():
            out[g] = x[i]
        del region
    return out


def _random_case(rng, shape, seed_frac=0.05):
    vol = rng.random(shape).astype(np.float32) * 0.3
    seeds = np.zeros(shape, np.uint8)
    u = rng.random(shape)
    seeds[u < seed_frac] = 1
    seeds[(u >= seed_frac) & (u < 2 * seed_frac)] = 2
    return vol, seeds


@pytest.mark.parametrize("shape,brick", [((9, 8, 7), (4, 4, 4)), ((13, 11), (5, 4)), ((6, 7, 5), (6, 7, 5))])
def test_block_pcg_matches_direct_solve(rng, shape, brick):
    vol, seeds = _random_case(rng, shape)
    whole = brick == shape
    bound = None if whole else rng.random(shape)
    got = rw.solve_level(vol, seeds, brick, bound, TIGHT).prob
    want = direct_brick_solve(vol, seeds, brick, bound)
    np.testing.assert_allclose(got, want, atol=1e-9, rtol=0)


def test_threaded_slabs_equal_serial(rng):
    vol, seeds = _random_case(rng, (20, 9, 10))
    bound = rng.random(vol.shape)
    a = rw.solve_level(vol, seeds, (4, 4, 4), bound, TIGHT).prob
    b = rw.solve_level_threaded(vol, seeds, (4, 4, 4), bound, TIGHT, workers=3).prob
    np.testing.assert_allclose(a, b, atol=1e-11, rtol=0)
    c = rw.solve_level_threaded(vol, seeds, (4, 4, 4), bound, TIGHT, workers=12).prob  # 5 x 2 tiles
    np.testing.assert_allclose(a, c, atol=1e-11, rtol=0)


def test_probabilities_bounded_and_seeds_exact():
    vol = syn.phantom((24, 24, 24))
    seeds = syn.seeds(vol.shape, "S1")
    res = rw.hierarchical_random_walker(vol, seeds, (8, 8, 8), levels=2, params=TIGHT)
    for p, s in zip(res.prob, res.seeds):
        assert p.min() >= -1e-9 and p.max() <= 1 + 1e-9
        assert np.all(p[s == 1] == 1.0) and np.all(p[s == 2] == 0.0)


def test_label_swap_symmetry():
    vol = syn.phantom((32, 40))
    seeds = syn.seeds(vol.shape, "S2")
    swapped = np.where(seeds == 1, 2, np.where(seeds == 2, 1, 0)).astype(np.uint8)
    a = rw.hierarchical_random_walker(vol, seeds, (8, 8), levels=3, params=TIGHT).prob[0]
    b = rw.hierarchical_random_walker(vol, swapped, (8, 8), levels=3, params=TIGHT).prob[0]
    np.testing.assert_allclose(a + b, 1.0, atol=1e-8)


def test_maximum_principle_whole_level(rng):
    # a harmonic function has no interior extrema: every unknown lies within
    # the range of its neighbours
    vol, seeds = _random_case(rng, (10, 10, 10), 0.02)
    p = rw.solve_level(vol, seeds, vol.shape, None, TIGHT).prob
    unk = seeds == 0
    pad = np.pad(p, 1, mode="edge")
    nbmax = np.full(p.shape, -np.inf)
    nbmin = np.full(p.shape, np.inf)
    for k in range(3):
        for s in (-1, 1):
            sl = [slice(1, -1)] * 3
            sl[k] = slice(1 + s, p.shape[k] + 1 + s)
            v = pad[tuple(sl)]
            nbmax = np.maximum(nbmax, v)
            nbmin = np.minimum(nbmin, v)
    assert np.all(p[unk] <= nbmax[unk] + 1e-9) and np.all(p[unk] >= nbmin[unk] - 1e-9)


def test_coarse_to_fine_reduces_to_single_level_when_one_level():
    vol = syn.phantom((20, 20, 20))
    seeds = syn.seeds(vol.shape, "S1")
    h = rw.hierarchical_random_walker(vol, seeds, (8, 8, 8), levels=1, params=TIGHT)
    s = rw.solve_level(vol, seeds, vol.shape, None, TIGHT)
    np.testing.assert_allclose(h.prob[0], s.prob, atol=0)


def test_zero_rhs_brick_is_exactly_zero():
    vol = np.zeros((4, 4), np.float32)
    seeds = np.zeros((4, 4), np.uint8)
    seeds[0, :] = 2
    p = rw.solve_level(vol, seeds, (4, 4), None, TIGHT).prob
    assert np.all(p == 0.0)


def test_seed_projection_rule():
    s = np.zeros((4, 5), np.uint8)
    s[0, 0] = 1            # block (0,0): fg only
    s[0, 2], s[1, 3] = 1, 2  # block (0,1): conflict -> 0
    s[3, 4] = 2            # ragged tail block (1,2): bg
    np.testing.assert_array_equal(rw.project_seeds(s), [[1, 0, 0], [0, 0, 2]])


def test_upsample_taps_and_clamp():
    parent = np.array([0.0, 4.0, 8.0])
    np.testing.assert_allclose(rw.upsample_linear(parent, (6,)), [0.0, 1.0, 3.0, 5.0, 7.0, 8.0])
    np.testing.assert_allclose(rw.upsample_linear(parent, (5,)), [0.0, 1.0, 3.0, 5.0, 7.0])


@pytest.mark.parametrize("name", ["h2d_s1", "h2d_s2"])
def test_oracle_reproduces_frozen_fixture(name):
    meta = MANIFEST["rw"][name]
    shape = tuple(meta["shape"])
    vol = syn.phantom(shape)
    seeds = syn.seeds(shape, meta["seeds"])
    res = rw.hierarchical_random_walker(vol, seeds, tuple(meta["brick"]), meta["levels"],
                                        rw.RWParams(tol=meta["tol"], max_iter=20000))
    g = load_golden(f"rw_{name}.npz")
    np.testing.assert_array_equal(res.prob[0].astype(np.float32), g["prob0"])
    np.testing.assert_array_equal(res.labels, g["labels"])


def test_brick_skip_rule_oracle():
    """decided_bricks: a brick is decided when the parent over it and its one-voxel halo is within
    eps of 0 or 1 (seeds count as decided); skipped bricks keep the upsampled parent."""
    bound = np.zeros((16, 16))
    seeds = np.zeros((16, 16), np.uint8)
    bound[3, 3] = 0.5           # inside brick (0, 0)
    bound[8, 2] = 0.01          # row 8 = halo of brick (0, 0) and inside brick (1, 0)
    seeds[12, 12] = 1
    bound[12, 12] = 0.5         # seeded: decided anyway
    d = rw.decided_bricks(bound, seeds, (8, 8), 1e-3)
    assert d.tolist() == [False, True, False, True]
    assert rw.decided_bricks(bound, seeds, (8, 8), 0.6).all()
    vol = syn.phantom((48, 40))
    sd = syn.seeds(vol.shape, "S1")
    full = rw.hierarchical_random_walker(vol, sd, (8, 8), 3, rw.RWParams(tol=1e-10))
    skip = rw.hierarchical_random_walker(vol, sd, (8, 8), 3, rw.RWParams(tol=1e-10), skip_eps=1e-6)
    assert np.abs(full.prob[0] - skip.prob[0]).max() < 1e-4


def _independent_projection(s):
    """Seed projection restated: a coarse voxel is fg (bg) when some child is fg
    (bg) and none is bg (fg); otherwise unseeded.  Ragged tails pad with unseeded children."""
    s = np.asarray(s)
    pad = [(0, n % 2) for n in s.shape]
    p = np.pad(s, pad)
    shape = []
    for n in p.shape:
        shape += [n // 2, 2]
    blocks = p.reshape(shape)
    axes = tuple(range(1, 2 * s.ndim, 2))
    fg, bg = (blocks == 1).any(axis=axes), (blocks == 2).any(axis=axes)
    return np.where(fg & ~bg, 1, np.where(bg & ~fg, 2, 0)).astype(np.uint8)


def _independent_upsample(parent, fine_shape):
    """Cell-centred linear prolongation restated with np.interp, one axis at a time: fine voxel g
    sits at parent coordinate g / 2 - 1/4, clamped to the parent's end values."""
    out = np.asarray(parent, np.float64)
    for dim, n in enumerate(fine_shape):
        c = np.arange(n) / 2.0 - 0.25
        out = np.apply_along_axis(lambda v: np.interp(c, np.arange(v.size), v), dim, out)
    return out


@pytest.mark.parametrize("shape,brick,levels", [((24, 20), (8, 8), 2), ((12, 10, 9), (4, 4, 4), 2),
                                                ((30, 26), (8, 8), 3)])
def test_hierarchy_matches_independent_composition(rng, shape, brick, levels):
    """The hierarchical driver (coarsest level whole; finer levels brick by brick from the upsampled
    parent) against the same chain assembled from independent pieces: the LOD pyramid pinned to the
    reference, restated seed projection and prolongation, and SuperLU per brick."""
    from oracle import lod

    vol = (rng.random(shape) * 0.3).astype(np.float32)
    vol[tuple(slice(0, n // 2) for n in shape)] += 0.5  # a blob, so levels differ
    seeds = np.zeros(shape, np.uint8)
    u = rng.random(shape)
    seeds[u < 0.04] = 1
    seeds[(u >= 0.04) & (u < 0.08)] = 2
    res = rw.hierarchical_random_walker(vol, seeds, brick, levels, TIGHT)
    vols = lod.lod_chain(vol, brick, levels)
    sl = [seeds]
    for _ in range(levels - 1):
        sl.append(_independent_projection(sl[-1]))
    for k in range(levels):
        np.testing.assert_array_equal(res.seeds[k], sl[k])
    prob = direct_brick_solve(vols[-1], sl[-1], vols[-1].shape, None)
    np.testing.assert_allclose(res.prob[-1], prob, atol=1e-8, rtol=0)
    for k in range(levels - 2, -1, -1):
        bound = _independent_upsample(prob, vols[k].shape)
        prob = direct_brick_solve(vols[k], sl[k], brick, bound)
        np.testing.assert_allclose(res.prob[k], prob, atol=1e-8, rtol=0)
