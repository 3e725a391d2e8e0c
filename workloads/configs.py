"""The five BASELINE.json workloads (+ small parametric ones for tests).

Readings of the paper applied here:
  R2  V(5,5) sweeps ("five pre- and post-smoothing steps").
  R3  omega = 1/3 (2D elementwise), 2/15 (3D elementwise), 1/6 (2D patch),
      1/18 (3D patch).
  R4  coarse p=1 solve: dense direct for config 1 ("direct solver,
      if the system is small"), CG + undamped elementwise AS to 1e-12 otherwise
      (PAPER.md:343).
  R6  outer flexible CG to relative residual < 1e-10 (BASELINE.json configs).
  R7  u = 0 strongly on Dirichlet box faces (bitmask bit 2*axis+side).
  R10 tensor space for configs 1,2,3,5; trunk space for config 4.
Only constants and recipes -- no method arithmetic.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field


@dataclass(frozen=True)
class Config:
    name: str
    dim: int
    n: int                      # cells per axis
    p: int                      # polynomial order
    space: str = "tensor"       # "tensor" | "trunk"
    physics: str = "poisson"    # "poisson" | "elasticity"
    alpha: float = 1e-8         # fictitious stiffness factor
    depth: int = 3              # space-tree integration depth
    geometry: dict = field(default_factory=lambda: {"kind": "none"})
    dirichlet: int = -1         # face bitmask; -1 = all faces
    traction_face: int = -1     # face index (2*axis+side) with traction (1,0,0); -1 none
    block: str = "element"      # "element" | "patch"
    omega: float | None = None  # None -> paper's value for (dim, block)
    n_pre: int = 5
    n_post: int = 5
    coarse: str = "as_pcg"      # "direct" | "as_pcg" | "jacobi_pcg"
    coarse_rtol: float = 1e-12
    coarse_maxit: int = 10000
    rtol: float = 1e-10
    maxit: int = 500
    E: float = 1.0
    nu: float = 0.3
    kmax: int = 0               # multi-level hp refinement depth (0 = uniform grid)
    refine: str = "cut"         # which elements are refined while depth < kmax: "cut" | "all"

    @property
    def n_f(self) -> int:
        return self.dim if self.physics == "elasticity" else 1

    @property
    def dirichlet_mask(self) -> int:
        return (1 << (2 * self.dim)) - 1 if self.dirichlet < 0 else self.dirichlet

    @property
    def omega_value(self) -> float:
        if self.omega is not None:
            return self.omega
        # PAPER.md:300
        table = {(2, "element"): 1.0 / 3.0, (3, "element"): 2.0 / 15.0,
                 (2, "patch"): 1.0 / 6.0, (3, "patch"): 1.0 / 18.0}
        return table[(self.dim, self.block)]

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    "cfg1": Config("cfg1", dim=2, n=16, p=3,
                   geometry={"kind": "explicit", "centres": [[0.503, 0.497]], "radii": [0.23]},
                   coarse="direct"),
    "cfg2": Config("cfg2", dim=3, n=32, p=2,
                   geometry={"kind": "seeded", "count": 8, "r_min": 0.05, "r_max": 0.12, "seed": 2}),
    "cfg3": Config("cfg3", dim=3, n=64, p=4, block="patch",
                   geometry={"kind": "seeded", "count": 64, "r_min": 0.03, "r_max": 0.08, "seed": 3}),
    # configs 4 and 5 name no coarse solver (4) or a Jacobi-PCG whose 750-900 inner iterations per
    # V-cycle dominate the solve (5); their default is the h-coarsened coarse CG (R21, P:227
    # Remark): config 4 2.02 s vs 8.66 s with CG+AS (profiles/r02_s3_bench_cfg4_*.json)
    "cfg4": Config("cfg4", dim=3, n=64, p=3, space="trunk", physics="elasticity",
                   geometry={"kind": "seeded", "count": 200, "r_min": 0.02, "r_max": 0.05, "seed": 4},
                   dirichlet=0b000001, traction_face=1, coarse="gmg_pcg"),
    "cfg5": Config("cfg5", dim=3, n=256, p=3,
                   geometry={"kind": "seeded", "count": 1000, "r_min": 0.01, "r_max": 0.03, "seed": 5},
                   coarse="gmg_pcg"),
}


def hp_plate(n: int, k: int, p: int = 2, block: str = "patch", **kw) -> Config:
    """The perforated linear-elastic plate of PAPER.md:709-713 (Sec. 4.2) on a multi-level hp
    grid ("elements that are intersected by the immersed boundary are refined
    recursively to a predefined depth"), scaled from l = 4 to the unit square (2D elasticity is
    scale-invariant): four circular cavities r = 0.3 sqrt(2) / 4 centred at (0.25 | 0.75)^2
    (reading R28: the figure is not reproduced in the text), E = 2.069e5, nu = 0.29, clamped at
    x = 0 (strong, R7), traction (1, 0) on x = 1 (R8), alpha = 1e-8, n = 1/h cells per axis."""
    r = 0.3 * 2 ** 0.5 / 4
    geom = {"kind": "explicit", "centres": [[0.25, 0.25], [0.75, 0.25], [0.25, 0.75], [0.75, 0.75]],
            "radii": [r] * 4}
    kw.setdefault("coarse", "direct")
    return Config(f"hp_plate_n{n}_k{k}_p{p}_{block}", dim=2, n=n, p=p, physics="elasticity",
                  geometry=geom, dirichlet=0b0001, traction_face=1, block=block, kmax=k,
                  E=2.069e5, nu=0.29, **kw)


def get_config(name: str) -> Config:
    return CONFIGS[name]


def small_config(dim=3, n=4, p=2, space="tensor", physics="poisson", voids=None,
                 seed=0, **kw) -> Config:
    """A small parametric workload for tests.  voids: None (no voids), an int
    (seeded count with radii in [0.08, 0.2]) or explicit (centres, radii)."""
    if voids is None:
        geom = {"kind": "none"}
    elif isinstance(voids, int):
        geom = {"kind": "seeded", "count": voids, "r_min": 0.08, "r_max": 0.2, "seed": seed}
    else:
        c, r = voids
        geom = {"kind": "explicit", "centres": [list(map(float, x)) for x in c],
                "radii": [float(x) for x in r]}
    if physics == "elasticity":
        kw.setdefault("dirichlet", 0b000001)
        kw.setdefault("traction_face", 1)
    return Config(f"small_d{dim}_n{n}_p{p}_{space}_{physics}", dim=dim, n=n, p=p, space=space,
                  physics=physics, geometry=geom, **kw)


def window_config(cfg: Config, k: int, corner=None) -> Config:
    """A bounded spatial SAMPLE of a workload (for the CPU-oracle timing legs of bench.py):
    the k^d cells of `cfg` starting at cell `corner` (default: the k^d window holding the most
    void volume near the domain centre), rescaled to [0,1]^d with k cells per axis -- same p,
    space, physics, smoother and solver constants, the voids that touch the window mapped by
    x -> (x - corner h) / (k h), u = 0 on the window faces.  No method arithmetic."""
    from .voids import config_voids
    import numpy as np
    c, r = config_voids(cfg)
    h = 1.0 / cfg.n
    d = cfg.dim
    if corner is None:
        mid = (cfg.n - k) // 2
        best, corner = -1.0, (mid,) * d
        for off in range(-(cfg.n // 4), cfg.n // 4 + 1, max(1, k // 2)):
            cand = tuple(min(max(mid + off, 0), cfg.n - k) for _ in range(d))
            lo = np.array(cand) * h
            hi = lo + k * h
            near = np.clip(c, lo, hi)
            touch = np.sum((c - near) ** 2, axis=1) < r ** 2
            vol = float(np.sum(r[touch] ** d))
            if vol > best:
                best, corner = vol, cand
    lo = np.array(corner, dtype=np.float64) * h
    hi = lo + k * h
    near = np.clip(c, lo, hi)
    touch = np.sum((c - near) ** 2, axis=1) < r ** 2
    cs = (c[touch] - lo) / (k * h)
    rs = r[touch] / (k * h)
    geom = {"kind": "explicit", "centres": cs.tolist(), "radii": rs.tolist()}
    return dataclasses.replace(cfg, name=f"{cfg.name}_window{k}", n=k, geometry=geom)
