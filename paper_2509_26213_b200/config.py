"""Random-walker parameters (canonically encodable, so they can feed operator ids).

The reference's operator params must be encodable by `canon.encode`
(dict/list/float/int/str only, `pkg/src/chunkcast/canon.py:19-50`); `params()`
returns that form.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass


@dataclass(frozen=True)
class RWConfig:
    beta: float = 100.0        # edge weight exp(-beta * dI^2), intensities in [0, 1]
    min_weight: float = 1e-6   # lower clamp of every edge weight
    tol: float = 1e-6          # per-brick ||r|| <= tol * ||b|| on the Jacobi-scaled system
    max_iter: int = 10_000     # per-brick iteration cap
    check_every: int = 16      # CG iterations per convergence poll (one CUDA graph)
    use_graph: bool = True     # streaming solver: run each poll interval as one CUDA graph launch
    resident: bool = True      # 32^3 bricks: solve each brick on chip (4-CTA cluster by default) instead of streaming
    cooperative: bool = True   # whole-level Jacobi-PCG (multigrid=False): one cooperative kernel for all iterations
    multigrid: bool | None = None  # whole-level solves: V-cycle-preconditioned CG (one cooperative kernel);
                               # None: on levels of >= 2^19 voxels, True: always, False: Jacobi-PCG
    coarse: bool = True        # 32^3 bricks (4-CTA engine): Jacobi + 8^3-aggregate coarse correction (False: Jacobi-PCG)
    skip_eps: float | None = None  # optional brick-skip rule (oracle/rw.py decided_bricks): bricks whose
                               # upsampled parent (+ halo) is within skip_eps of 0 or 1 are not solved
    fused_setup: bool = True   # build the brick system with the fused per-brick setup kernel
    cluster: int = 4           # resident solver: CTAs per brick cluster (4: weights in TMEM, default; 8: all in registers;
                               # 16: 2 CTAs/SM; 512: 8-CTA with 512 threads) — 4 is 1.4x faster than 8 on config 4

    def params(self) -> dict:
        d = asdict(self)
        d.pop("check_every")
        d.pop("use_graph")
        d.pop("resident")
        d.pop("cooperative")
        d.pop("multigrid")
        d.pop("coarse")
        d.pop("cluster")
        d.pop("fused_setup")
        skip = d.pop("skip_eps")
        out = {k: (float(v) if isinstance(v, float) else int(v)) for k, v in d.items()}
        if skip is not None:  # part of the result's identity only when the rule is on
            out["skip_eps"] = float(skip)
        return out
