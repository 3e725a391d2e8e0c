"""Shared test helpers for the multi-level hp path: map the native generator's DOF keys onto the
oracle's numbering (no method arithmetic)."""
import numpy as np


def key_perm(P, keys):
    """perm[i] = oracle DOF index of library DOF i (keys: int32 [ndof, 8] from fcm_hp_disc_keys)."""
    d = P.cfg.dim
    okeys = {}
    for i, (k, c) in enumerate(P.keys):
        j, X, dg = k[0], k[1:1 + d], k[1 + d:1 + 2 * d]
        okeys[(j,) + tuple(X) + (0,) * (3 - d) + tuple(dg) + (0,) * (3 - d) + (c,)] = i
    perm = np.array([okeys[tuple(int(v) for v in r)] for r in keys], dtype=np.int64)
    assert len(np.unique(perm)) == len(perm) == P.ndof
    return perm


HP_CASES = {
    # name: (config factory kwargs)
    "plate_n8_k2_patch": dict(kind="plate", n=8, k=2, block="patch"),
    "plate_n8_k3_element": dict(kind="plate", n=8, k=3, block="element"),
    "poisson2d_p3_k2_patch": dict(kind="small", dim=2, n=3, p=3, k=2, block="patch"),
    "poisson2d_p2_k2_element_aspcg": dict(kind="small", dim=2, n=4, p=2, k=2, block="element", coarse="as_pcg"),
    "poisson3d_p2_k1_patch": dict(kind="small", dim=3, n=3, p=2, k=1, block="patch"),
    "elast3d_p2_k1_element": dict(kind="small", dim=3, n=3, p=2, k=1, block="element", physics="elasticity"),
    # every base element cut and refined: (1,0) is empty and dropped (degenerate case)
    "poisson2d_fully_refined": dict(kind="small", dim=2, n=2, p=2, k=1, block="patch", void=([[0.5, 0.5]], [0.3])),
}


def hp_config(name):
    from workloads import hp_plate, small_config
    c = dict(HP_CASES[name])
    if c.pop("kind") == "plate":
        return hp_plate(c["n"], c["k"], block=c["block"])
    dim = c["dim"]
    void = c.get("void") or (([[0.45] * dim], [0.28]) if dim == 2 else ([[0.3] * dim], [0.15]))
    kw = {"block": c["block"], "coarse": c.get("coarse", "direct")}
    phys = c.get("physics", "poisson")
    if phys == "poisson":
        kw["dirichlet"] = 0b0101 if dim == 2 else 0b000101
    return small_config(dim, c["n"], c["p"], physics=phys, voids=void, kmax=c["k"], **kw)
