"""CPU oracle for the hierarchical random-walker hot path — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg
(`--impl reference` and the `cpu_baseline` field) may import anything from
here, and only as the checker / the timed CPU reference.  The product package
`paper_2509_26213_b200` never imports this package; its device path fails
loudly when the CUDA library is missing instead of falling back to the CPU.

Contents
--------
* `oracle.lod` — dense float64 restatement of the reference's LOD pyramid
  (`chunkcast.ops.separable_conv` + `downsample_mean` + `build_lod`,
  `pkg/src/chunkcast/ops.py:471-548, 611-676, 714-727`).  Pinned bit-exactly
  against the reference itself: `tests/golden/make_golden.py` imports
  `chunkcast` from `/root/reference/pkg/src` and freezes its outputs, and the
  reference's own known-answer tests (`pkg/tests/test_operators.py:418-484`)
  are replayed in `tests/test_oracle_lod.py`.
* `oracle.rw` — the random walker (edge weights, seed projection, coarse→fine
  upsampling, block-diagonal Jacobi-PCG in float64, hierarchical driver,
  labels).  **RW parity is unpinned against the reference**: the reference
  repository contains no random-walker code (`SPEC.md:8, 425, 802`); the
  algorithm is restated from Grady 2006 (cited at `PAPER.md:159`) and Drees
  et al. 2022 (cited at `PAPER.md:419`).  The restatement is instead pinned
  against an independent direct sparse solve (`scipy.sparse.linalg.spsolve`
  on an explicitly assembled Laplacian, `tests/test_oracle_rw.py`).
"""
