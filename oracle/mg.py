"""Hierarchical p-multigrid with additive Schwarz smoothing (oracle).
TEST INFRASTRUCTURE ONLY.

Level operators ("A_{l-1} = R_l A_l R_l^T", P:209-216 hierarchical
matrices): A_q = A[I_q, I_q], I_q = DOFs of mode order <= q; R = [I 0] is index
selection.  Levels: arithmetic p-sequence p, p-1, ..., 1.

Additive Schwarz (Eq. AdditiveSchwarz):
  M^{-1} = sum_i P_i (P_i^T A P_i)^{-1} P_i^T,
blocks: elementwise = the free level DOFs supported on one cell;
patchwise = the union over the 2^d cells around a grid vertex (every vertex,
boundary ones included; empty blocks skipped) -- patch_rule "closure", the DOFs
whose support intersects the patch, size (2p+1)^d as Table 1 prints;
patch_rule "interior" (reading R19, a variant kept only for the paper's
iteration-count pin) keeps the DOFs whose whole support lies inside the patch.  Block inverses by dense LU
(numpy.linalg.inv = LAPACK getrf/getri path, O8).  The sum is accumulated
serially in block order (cell / vertex index, x fastest).

V-cycle: Algorithm 1 with reading R1 (the residual is recomputed
before every smoothing sweep, P:124-126 fixed-point smoothing), x~ = 0 on
entry, n_s pre and post sweeps.
Coarse level: 'direct' dense LU; 'as_pcg' CG with the
undamped elementwise AS preconditioner at p = 1, x0 = 0, stop at
||r|| < rtol ||r0|| (reading R4); 'jacobi_pcg' the same with diag(A0); 'gmg_pcg'
the same CG preconditioned by one geometric V-cycle over h-coarsened p=1 grids
(P:227 Remark, class GeometricLevels, reading R21).
Outer solver: flexible (Polak-Ribiere) PCG, x0 = 0, stop at the recursive
||r_k||_2 / ||b||_2 < rtol (readings R5, R6).
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp


class Level:
    def __init__(self, prob, q, block, A_full, omega, inv_method="lu", patch_rule="closure"):
        dof = prob.dof
        self.q = q
        self.idx = dof.level_dofs(q)
        self.n = len(self.idx)
        self.A = A_full[self.idx][:, self.idx].tocsr()
        self.omega = omega
        pos = np.full(dof.ndof, -1, dtype=np.int64)
        pos[self.idx] = np.arange(self.n)
        mq = dof.level_m(q)
        cd = dof.cell_dofs[:, :mq]
        cfg = prob.cfg
        blocks = []
        if block == "element":
            for c in range(cd.shape[0]):
                g = cd[c][cd[c] >= 0]
                if len(g):
                    blocks.append(pos[g])
        else:  # patch: 2^d cells around each grid vertex
            n, d = cfg.n, cfg.dim
            if patch_rule == "interior":
                # number of cells in the support of each DOF (reading R19 variant)
                ok = cd >= 0
                nsup = np.bincount(cd[ok], minlength=dof.ndof)
            for v in range((n + 1) ** d):
                vc = [(v // (n + 1) ** a) % (n + 1) for a in range(d)]
                cells = []
                for corner in range(1 << d):
                    cc = [vc[a] - 1 + ((corner >> a) & 1) for a in range(d)]
                    if all(0 <= x < n for x in cc):
                        cells.append(sum(cc[a] * n ** a for a in range(d)))
                allg = np.concatenate([cd[c][cd[c] >= 0] for c in sorted(cells)])
                if patch_rule == "closure":
                    # every DOF whose support intersects the patch (Table 1: (2p+1)^d)
                    g = np.unique(allg)
                else:
                    # "interior": only DOFs whose whole support lies inside the patch
                    g, cnt = np.unique(allg, return_counts=True)
                    g = g[cnt == nsup[g]]
                if len(g):
                    blocks.append(pos[g])
        self.blocks = blocks
        self.inv = [None] * len(blocks)
        Ad = self.A
        by_size = {}
        for i, b in enumerate(blocks):
            by_size.setdefault(len(b), []).append(i)
        for size, ids in by_size.items():
            stack = np.stack([Ad[blocks[i]][:, blocks[i]].toarray() for i in ids])
            if inv_method == "lu":
                inv = np.linalg.inv(stack)
            else:   # "chol": a second backward-stable inverse, used only to measure the
                # rounding spread between two valid fp64 evaluations (reading R18)
                eye = np.eye(size)
                inv = np.stack([sla.cho_solve(sla.cho_factor(S, lower=True), eye) for S in stack])
            for k, i in enumerate(ids):
                self.inv[i] = inv[k]

    def set_blocks(self, blocks, inverses):
        """Replace this level's blocks and inverses by externally supplied ones (the identical-
        setup parity protocol: the GPU exports its inverses, the oracle's
        smoother then runs on the same setup data).  blocks: level-local index arrays."""
        self.blocks = [np.asarray(b, dtype=np.int64) for b in blocks]
        self.inv = [np.asarray(a, dtype=np.float64) for a in inverses]

    def schwarz(self, r):
        """M^{-1} r = sum_i P_i A_i^{-1} P_i^T r, accumulated serially in block order."""
        idx = np.concatenate(self.blocks)
        vals = np.concatenate([self.inv[i] @ r[b] for i, b in enumerate(self.blocks)])
        return np.bincount(idx, weights=vals, minlength=self.n)


def _vertex_dofs(n, dim, n_f, dmask):
    """Free p=1 DOFs of a vertex grid with n cells per axis, Dirichlet faces removed (R7), in
    the oracle's order (z, y, x slowest to fastest, then component).  Returns [N, dim+1]
    (positions per axis, component)."""
    import itertools
    out = []
    rng = []
    for a in range(dim):
        lo = 1 if (dmask >> (2 * a)) & 1 else 0
        hi = n - 1 if (dmask >> (2 * a + 1)) & 1 else n
        rng.append(range(lo, hi + 1))
    for pos in itertools.product(*reversed(rng)):
        pos = tuple(reversed(pos))
        for c in range(n_f):
            out.append(pos + (c,))
    return np.array(out, dtype=np.int64).reshape(-1, dim + 1)


class GeometricLevels:
    """h-coarsening of the p=1 level (PAPER.md:227 Remark: "the p=1, k=0 problem can be
    coarsened further using a standard geometric multigrid algorithm"), reading R21 of
    DESIGN.md: vertex grids n, n/2, n/4, ... (coarsen while n is even and n > 4), standard
    (bi/tri)linear interpolation P between nested vertex grids restricted to the free DOFs,
    Galerkin operators A_{i+1} = P^T A_i P (P:118's R A R^T with R = P^T), elementwise additive
    Schwarz on every level (blocks = the free DOFs of one cell of that level's grid, assembled
    A_i sub-blocks, dense inverses, omega of P:300), V(n_pre, n_post) cycles of Algorithm 1's
    form (R1), LU on the coarsest grid.  Level 0 is the p=1 level itself (its matrix A_1 and its
    elementwise blocks come from the caller)."""

    def __init__(self, cfg, A1, keys1, blocks0, inv0, omega, n_pre, n_post):
        d, n_f, p = cfg.dim, cfg.n_f, cfg.p
        per = (p + 1) ** 3 * n_f
        ent = keys1 // per
        comp = keys1 % n_f
        X = [(ent // (2 * cfg.n + 1) ** a) % (2 * cfg.n + 1) for a in range(d)]
        assert all(np.all(x % 2 == 0) for x in X), "level-1 DOFs are vertex DOFs"
        self.pos = [np.stack([x // 2 for x in X] + [comp], axis=1)]
        self.A = [A1.tocsr()]
        self.blocks = [blocks0]
        self.inv = [inv0]
        self.P = []
        self.n = [cfg.n]
        self.omega, self.n_pre, self.n_post = omega, n_pre, n_post
        n = cfg.n
        while n % 2 == 0 and n > 4:
            nc = n // 2
            cpos = _vertex_dofs(nc, d, n_f, cfg.dirichlet_mask)
            index = {tuple(r): i for i, r in enumerate(cpos.tolist())}
            rows, cols, vals = [], [], []
            for i, r in enumerate(self.pos[-1].tolist()):
                par = [[(r[a] // 2, 1.0)] if r[a] % 2 == 0 else [((r[a] - 1) // 2, 0.5), ((r[a] + 1) // 2, 0.5)]
                       for a in range(d)]
                import itertools
                for combo in itertools.product(*par):
                    key = tuple(c[0] for c in combo) + (r[d],)
                    j = index.get(key)
                    if j is not None:
                        rows.append(i)
                        cols.append(j)
                        vals.append(float(np.prod([c[1] for c in combo])))
            P = sp.csr_matrix((vals, (rows, cols)), shape=(len(self.pos[-1]), len(cpos)))
            Ac = (P.T @ self.A[-1] @ P).tocsr()
            # elementwise blocks of the coarse grid: the free DOFs of each cell
            blocks = []
            for cell in range(nc ** d):
                cc = [(cell // nc ** a) % nc for a in range(d)]
                ids = []
                for corner in range(1 << d):
                    v = tuple(cc[a] + ((corner >> a) & 1) for a in range(d))
                    for c in range(n_f):
                        j = index.get(v + (c,))
                        if j is not None:
                            ids.append(j)
                if ids:
                    blocks.append(np.array(sorted(ids), dtype=np.int64))
            inv = [np.linalg.inv(Ac[b][:, b].toarray()) for b in blocks]
            self.P.append(P)
            self.A.append(Ac)
            self.blocks.append(blocks)
            self.inv.append(inv)
            self.pos.append(cpos)
            self.n.append(nc)
            n = nc
        self.lu = sla.lu_factor(self.A[-1].toarray())

    def _schwarz(self, i, r):
        idx = np.concatenate(self.blocks[i])
        vals = np.concatenate([self.inv[i][k] @ r[b] for k, b in enumerate(self.blocks[i])])
        return np.bincount(idx, weights=vals, minlength=self.A[i].shape[0])

    def vcycle(self, b, i=0):
        """Geometric V-cycle on h-level i (x = 0 on entry; residual before every sweep, R1)."""
        if i == len(self.A) - 1:
            return sla.lu_solve(self.lu, b)
        A, w = self.A[i], self.omega
        x = np.zeros_like(b)
        for _ in range(self.n_pre):
            x = x + w * self._schwarz(i, b - A @ x)
        r = b - A @ x
        x = x + self.P[i] @ self.vcycle(self.P[i].T @ r, i + 1)
        for _ in range(self.n_post):
            x = x + w * self._schwarz(i, b - A @ x)
        return x


class Hierarchy:
    def __init__(self, prob, block=None, omega=None, n_pre=None, n_post=None, coarse=None,
                 coarse_rtol=None, coarse_maxit=None, inv="lu", patch_rule="closure"):
        cfg = prob.cfg
        self.prob = prob
        self.block = block or cfg.block
        if omega is None:
            omega = cfg.omega if cfg.omega is not None else cfg.replace(block=self.block).omega_value
        self.omega = omega
        self.n_pre = cfg.n_pre if n_pre is None else n_pre
        self.n_post = cfg.n_post if n_post is None else n_post
        self.coarse = coarse or cfg.coarse
        self.coarse_rtol = cfg.coarse_rtol if coarse_rtol is None else coarse_rtol
        self.coarse_maxit = cfg.coarse_maxit if coarse_maxit is None else coarse_maxit
        A = prob.A
        self.levels = {}
        for q in range(cfg.p, 0, -1):
            blk = self.block if q > 1 else "element"   # coarse AS is elementwise (R11)
            need_blocks = q > 1 or self.coarse in ("as_pcg", "gmg_pcg")
            if need_blocks:
                self.levels[q] = Level(prob, q, blk, A, self.omega if q > 1 else 1.0, inv_method=inv,
                                       patch_rule=patch_rule)
            else:
                lv = Level.__new__(Level)
                lv.q = q
                lv.idx = prob.dof.level_dofs(q)
                lv.n = len(lv.idx)
                lv.A = A[lv.idx][:, lv.idx].tocsr()
                self.levels[q] = lv
        # restriction selections: positions of I_{q-1} inside I_q
        self.sel = {}
        for q in range(cfg.p, 1, -1):
            self.sel[q] = np.searchsorted(self.levels[q].idx, self.levels[q - 1].idx)
        c = self.levels[1]
        if self.coarse == "direct":
            self.lu = sla.lu_factor(c.A.toarray())
        elif self.coarse == "jacobi_pcg":
            self.diag = c.A.diagonal()
        elif self.coarse == "gmg_pcg":
            # the level-1 smoother of the h-hierarchy uses the ELEMENTWISE omega (R21)
            w_el = cfg.replace(block="element", omega=None).omega_value
            self.gmg = GeometricLevels(cfg, c.A, prob.dof.keys[c.idx], c.blocks, c.inv, w_el,
                                       self.n_pre, self.n_post)
        self.coarse_iters = []

    def set_coarse_inverse(self, inv):
        """Identical-setup parity protocol: apply an externally supplied
        dense A_1^{-1} as the direct coarse solve instead of this oracle's own LU."""
        self.coarse_inv = np.asarray(inv, dtype=np.float64)

    # -- coarse level --------------------------------------
    def coarse_solve(self, b):
        lv = self.levels[1]
        if self.coarse == "direct":
            if getattr(self, "coarse_inv", None) is not None:
                return self.coarse_inv @ b
            return sla.lu_solve(self.lu, b)
        if self.coarse == "gmg_pcg":
            prec = self.gmg.vcycle
        elif self.coarse == "as_pcg":
            prec = lv.schwarz
        else:
            prec = lambda r: r / self.diag  # noqa: E731
        x, it = pcg(lambda v: lv.A @ v, b, prec, self.coarse_rtol, self.coarse_maxit,
                    rel_to="r0")
        self.coarse_iters.append(it)
        return x

    # -- Algorithm 1 -------------------------------------------------
    def vcycle(self, b, q=None):
        if q is None:
            q = self.prob.cfg.p
        if q == 1:
            return self.coarse_solve(b)
        lv = self.levels[q]
        A = lv.A
        w = self.omega
        x = np.zeros(lv.n)
        for _ in range(self.n_pre):            # pre-smoothing, residual per sweep (R1)
            r = b - A @ x
            x = x + w * lv.schwarz(r)
        r = b - A @ x                           # update residual
        e = self.vcycle(r[self.sel[q]], q - 1)  # r_{l-1} = R r_l
        x[self.sel[q]] += e                     # x += R^T e
        for _ in range(self.n_post):           # P:169 residual, then post-smoothing
            r = b - A @ x
            x = x + w * lv.schwarz(r)
        return x

    def mg_solve(self, b, rtol=None, maxit=None):
        """Multigrid as a stand-alone solver: x_0 = 0,
        x_i = x_{i-1} + V(b - A x_{i-1}); stop when ||b - A x_i|| / ||b|| < rtol (strict) or
        after maxit V-cycles.  Returns x, i, [||r_0||/||b||, ..., ||r_i||/||b||]; the contraction
        numbers rho_i (Eq. contraction) are hist[1:] / hist[:-1]."""
        cfg = self.prob.cfg
        rtol = cfg.rtol if rtol is None else rtol
        maxit = cfg.maxit if maxit is None else maxit
        A = self.levels[cfg.p].A
        nb = np.linalg.norm(b)
        x = np.zeros_like(b)
        if nb == 0:
            return x, 0, [0.0]
        r = b.copy()
        hist = [1.0]
        it = 0
        while it < maxit:
            x = x + self.vcycle(r)
            r = b - A @ x
            it += 1
            hist.append(np.linalg.norm(r) / nb)
            if hist[-1] < rtol:
                break
        return x, it, hist

    def fcg(self, b, rtol=None, maxit=None, force_iters=None, callback=None):
        cfg = self.prob.cfg
        rtol = cfg.rtol if rtol is None else rtol
        maxit = cfg.maxit if maxit is None else maxit
        A = self.levels[cfg.p].A
        return fcg(lambda v: A @ v, b, self.vcycle, rtol, maxit, force_iters=force_iters,
                   callback=callback)


def pcg(apply_A, b, prec, rtol, maxit, rel_to="b"):
    """Standard preconditioned CG, x0 = 0 (coarse solver)."""
    x = np.zeros_like(b)
    r = b.copy()
    nr0 = np.linalg.norm(r)
    if nr0 == 0.0:
        return x, 0
    z = prec(r)
    p = z.copy()
    rz = r @ z
    it = 0
    while it < maxit:
        q = apply_A(p)
        pq = p @ q
        if pq <= 0:
            raise FloatingPointError("p^T A p <= 0 in coarse CG")
        a = rz / pq
        x += a * p
        r -= a * q
        it += 1
        if np.linalg.norm(r) < rtol * nr0:
            break
        z = prec(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it


def fcg(apply_A, b, prec, rtol, maxit, force_iters=None, callback=None):
    """Flexible (Polak-Ribiere) PCG, x0 = 0 (R5/R6).
    Returns (x, iterations, relative residual history [||r_k||/||b||]).
    callback(k, x_k), if given, sees every iterate (test bookkeeping only)."""
    x = np.zeros_like(b)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return x, 0, [0.0]
    r = b.copy()
    z = prec(r)
    p = z.copy()
    rz = r @ z
    hist = [1.0]
    it = 0
    while True:
        q = apply_A(p)
        pq = p @ q
        if pq <= 0:
            raise FloatingPointError("p^T A p <= 0 in FCG")
        a = rz / pq
        x = x + a * p
        r_old = r
        r = r - a * q
        it += 1
        hist.append(np.linalg.norm(r) / nb)
        if callback is not None:
            callback(it, x)
        if force_iters is not None:
            if it >= force_iters:
                break
        elif hist[-1] < rtol or it >= maxit:
            break
        z = prec(r)
        rz_new = r @ z
        beta = (rz_new - z @ r_old) / rz
        p = z + beta * p
        rz = rz_new
    return x, it, hist
