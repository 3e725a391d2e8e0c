"""Multi-level hp-refinement and the hp-multigrid on it (oracle).  TEST INFRASTRUCTURE ONLY.

PAPER.md:99-102 (Sec. 2.2): "spatial refinement is performed by superposing a base element with
subelements formed by uniform bisections ... recursively until the desired refinement depth";
"the deactivation of specific topological components following a simple rule-set ensures
compatibility and linear independence" (Fig. 2 caption, rule set deferred to [Zander2016]).
P:207: "in the case of multi-level hp-grids, it is required to first reduce the polynomial order
p in the overlay meshes, before reducing the levels of refinement"; P:217 + Fig. hpmultigrid
(P:219-224): levels (p,k), (p-1,k), ..., (1,k), (1,k-1), ..., (1,0); Remark P:226: (1,0) is the
coarsest level.  Blocks (Fig. 7): elementwise = all basis functions supported on an
element, patchwise = all basis functions supported on the base elements around a base vertex.

Readings:
  R25 activation rule.  A level-j entity (vertex / edge / face / cell interior of the level-j
      grid, doubled coordinates X as in dofmap.py) is ACTIVE iff
        (compatibility) j = 0, or every level-j element adjacent to it inside the domain exists
        (the entity is not on the boundary of the level-j overlay region, so every overlay
        function vanishes on that boundary), and
        (independence) at least one existing adjacent level-j element is a LEAF (an entity owned
        only by refined elements is represented by the finer overlay instead).
      Pinned by: independence (SPD mass matrix), C0 traces across every leaf interface, exact
      reproduction of global polynomials of degree p, and identity of the space with the uniform
      fine grid when every element is refined.
  R26 blocks: "this selection is performed on the granularity of the base elements ... and
      node-based element patches for multi-level hp-grids" (Fig. 7 caption): an
      elementwise block is the set of level DOFs nonzero on one BASE element (overlay functions
      included), a patchwise block those nonzero on the 2^d base elements around a base vertex;
      so a function lies in at most 2^d elementwise blocks (n_max of P:298 as on uniform
      grids).  Empty blocks are skipped; identical blocks are one block (a block is a set).
  R27 2D elasticity: plane strain (the d-dimensional isotropic law of quadrature.py).
Dirichlet (R7): every DOF of an entity on a Dirichlet box face is eliminated.  Tensor space.
Quadrature per leaf: the space tree of quadrature.py (depth cfg.depth below the LEAF, (p+1)^d
Gauss points per sub-box); every ancestor's functions are polynomials of degree <= p on a leaf.
"""
from __future__ import annotations

import itertools

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import basis, geometry, quadrature
from .mg import fcg, pcg


def _nodal_X(idx_a, k):
    """Doubled coordinate of 1D mode k of the cell with index idx_a (dofmap.py convention)."""
    return 2 * idx_a + (0 if k == 0 else 2 if k == 1 else 1)


class Mesh:
    """Base grid n^d on [0,1]^d plus refinement trees."""

    def __init__(self, cfg, centres, radii, refine=None):
        self.cfg = cfg
        dim, n, kmax = cfg.dim, cfg.n, cfg.kmax
        self.dim, self.n, self.kmax = dim, n, kmax
        self.refined = {}
        stack = [(0, idx) for idx in itertools.product(range(n), repeat=dim)]
        while stack:
            j, idx = stack.pop()
            h = 1.0 / (n * 2 ** j)
            lo = np.array(idx, dtype=np.float64) * h
            if j >= kmax:
                ref = False
            elif refine is not None:
                ref = bool(refine(j, idx))
            elif cfg.refine == "all":
                ref = True
            else:   # elements intersected by the immersed boundary are refined
                ref = geometry.classify_box(lo, lo + h, centres, radii) == geometry.CUT
            self.refined[(j, idx)] = ref
            if ref:
                for c in itertools.product((0, 1), repeat=dim):
                    stack.append((j + 1, tuple(2 * i + ca for i, ca in zip(idx, c))))
        self.elements = sorted(self.refined, key=lambda e: (e[0], e[1][::-1]))
        self.leaves = [e for e in self.elements if not self.refined[e]]
        self._act = {}

    def h(self, j):
        return 1.0 / (self.n * 2 ** j)

    def adjacent(self, j, X):
        N = self.n * 2 ** j
        rng = []
        for x in X:
            if x % 2:
                rng.append([(x - 1) // 2])
            else:
                rng.append([i for i in (x // 2 - 1, x // 2) if 0 <= i < N])
        return [tuple(e) for e in itertools.product(*rng)]

    def active(self, j, X):
        """Reading R25."""
        key = (j, X)
        if key not in self._act:
            adj = self.adjacent(j, X)
            ex = [e for e in adj if (j, e) in self.refined]
            ok = (j == 0 or len(ex) == len(adj)) and any(not self.refined[(j, e)] for e in ex)
            self._act[key] = ok
        return self._act[key]

    def ancestors(self, e):
        """(j, idx) of e and all its ancestors, base element first."""
        j, idx = e
        return [(i, tuple(x >> (j - i) for x in idx)) for i in range(j + 1)]


class MlhpProblem:
    """Discrete system of a multi-level hp finite cell problem: DOF map with level tags
    (mode order q, refinement depth j), leaf element matrices over the superposed basis, global
    CSR matrix and load.  Duck-types what MlhpHierarchy needs."""

    def __init__(self, cfg, centres=None, radii=None, refine=None):
        from workloads import config_voids
        if centres is None:
            centres, radii = config_voids(cfg)
        self.cfg = cfg
        self.centres = np.asarray(centres, dtype=np.float64).reshape(-1, cfg.dim)
        self.radii = np.asarray(radii, dtype=np.float64).reshape(-1)
        self.mesh = M = Mesh(cfg, self.centres, self.radii, refine)
        dim, p, n_f = cfg.dim, cfg.p, cfg.n_f
        self.modes = basis.element_modes(dim, p, "tensor")
        self.mode_order = [basis.mode_order(m, "tensor") for m in self.modes]
        mask = cfg.dirichlet_mask
        keys = set()
        self._elem_funcs = {}
        for e in M.elements:
            j, idx = e
            N = M.n * 2 ** j
            fl = []
            for mi, mode in enumerate(self.modes):
                X = tuple(_nodal_X(idx[a], mode[a]) for a in range(dim))
                if not M.active(j, X):
                    continue
                dirich = False
                for a in range(dim):
                    if X[a] % 2 == 0:
                        if ((mask >> (2 * a)) & 1) and X[a] == 0:
                            dirich = True
                        if ((mask >> (2 * a + 1)) & 1) and X[a] == 2 * N:
                            dirich = True
                if dirich:
                    continue
                degs = tuple(mode[a] if mode[a] >= 2 else 0 for a in range(dim))
                fl.append((mi, (j,) + X + degs))
                keys.add((j,) + X + degs)
            self._elem_funcs[e] = fl
        skeys = sorted(keys)
        self.keys = [(k, c) for k in skeys for c in range(n_f)]
        self.ndof = len(self.keys)
        kpos = {k: i for i, k in enumerate(skeys)}
        self.dof_order = np.zeros(self.ndof, dtype=np.int64)
        self.dof_depth = np.zeros(self.ndof, dtype=np.int64)
        for i, (k, c) in enumerate(self.keys):
            degs = k[1 + dim:]
            self.dof_order[i] = max([1] + [d for d in degs if d >= 2])
            self.dof_depth[i] = k[0]
        # scalar functions of each element: (mode index, scalar key index)
        self.elem_funcs = {e: [(mi, kpos[k]) for mi, k in fl] for e, fl in self._elem_funcs.items()}
        # leaf DOF lists (global indices), matrices and loads
        self.leaf_dofs, self.leaf_K, self.leaf_f = [], [], []
        for leaf in M.leaves:
            d, K, f = self._leaf_system(leaf)
            self.leaf_dofs.append(d)
            self.leaf_K.append(K)
            self.leaf_f.append(f)
        rows, cols, vals = [], [], []
        self.b = np.zeros(self.ndof)
        for d, K, f in zip(self.leaf_dofs, self.leaf_K, self.leaf_f):
            rows.append(np.repeat(d, len(d)))
            cols.append(np.tile(d, len(d)))
            vals.append(K.ravel())
            np.add.at(self.b, d, f)
        self.A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                               shape=(self.ndof, self.ndof)).tocsr()

    # -- superposed basis on a leaf ("superposing a base element with subelements") --
    def leaf_functions(self, leaf):
        """Scalar functions nonzero on `leaf`: list of (ancestor element, mode index, scalar index)."""
        out = []
        for anc in self.mesh.ancestors(leaf):
            for mi, si in self.elem_funcs[anc]:
                out.append((anc, mi, si))
        return out

    def eval_functions(self, funcs, pts):
        """Values [nf, npts] and physical gradients [nf, npts, dim] at physical points."""
        dim = self.cfg.dim
        val = np.zeros((len(funcs), len(pts)))
        grad = np.zeros((len(funcs), len(pts), dim))
        for i, (anc, mi, _) in enumerate(funcs):
            j, idx = anc
            h = self.mesh.h(j)
            ref = 2.0 * (pts - np.array(idx, dtype=np.float64) * h) / h - 1.0
            v, g = basis.eval_element([self.modes[mi]], ref)
            val[i] = v[0]
            grad[i] = g[0] * (2.0 / h)
        return val, grad

    def _leaf_system(self, leaf):
        cfg = self.cfg
        dim, n_f, p = cfg.dim, cfg.n_f, cfg.p
        j, idx = leaf
        h = self.mesh.h(j)
        lo = np.array(idx, dtype=np.float64) * h
        funcs = self.leaf_functions(leaf)
        nfun = len(funcs)
        dofs = np.array([si * n_f + c for (_, _, si) in funcs for c in range(n_f)], dtype=np.int64)
        pts, ws, als = [], [], []
        for slo, shi, kind in quadrature.leaves(lo, lo + h, cfg.depth, self.centres, self.radii):
            _, phys, w = quadrature._leaf_points(slo, shi, lo, h, p + 1, dim)
            if kind == geometry.PHYS:
                a = np.ones(len(w))
            elif kind == geometry.FICT:
                a = np.full(len(w), cfg.alpha)
            else:
                a = np.where(geometry.point_is_fictitious(phys, self.centres, self.radii), cfg.alpha, 1.0)
            pts.append(phys)
            ws.append(w)
            als.append(a)
        pts, w, a = np.concatenate(pts), np.concatenate(ws), np.concatenate(als)
        val, G = self.eval_functions(funcs, pts)
        wa = w * a
        K = np.zeros((nfun * n_f, nfun * n_f))
        f = np.zeros(nfun * n_f)
        if cfg.physics == "poisson":
            Gf = G.reshape(nfun, -1)
            K += (Gf * np.repeat(wa, dim)[None, :]) @ Gf.T
            f += val @ wa
        else:
            lam, mu = quadrature.lame(cfg.E, cfg.nu)
            KK = K.reshape(nfun, n_f, nfun, n_f)
            dot = np.einsum("aqd,bqd,q->ab", G, G, wa)
            for i in range(n_f):
                for k in range(n_f):
                    KK[:, i, :, k] += (lam * np.einsum("aq,bq,q->ab", G[:, :, i], G[:, :, k], wa)
                                       + mu * np.einsum("aq,bq,q->ab", G[:, :, k], G[:, :, i], wa))
                KK[:, i, :, i] += mu * dot
        if cfg.traction_face >= 0:   # traction (1, 0[, 0]) on the face (R8), leaves touching it
            axis, side = cfg.traction_face // 2, cfg.traction_face % 2
            if (idx[axis] == (self.mesh.n * 2 ** j - 1) if side else idx[axis] == 0):
                xg, wg = basis.gauss(p + 1)
                others = [b for b in range(dim) if b != axis]
                fp, fw = [], []
                for combo in itertools.product(range(p + 1), repeat=dim - 1):
                    x = lo.copy()
                    x[axis] = lo[axis] + (h if side else 0.0)
                    wt = 1.0
                    for b, c in zip(others, combo):
                        x[b] = lo[b] + 0.5 * h * (xg[c] + 1.0)
                        wt *= 0.5 * h * wg[c]
                    fp.append(x)
                    fw.append(wt)
                fv, _ = self.eval_functions(funcs, np.array(fp))
                f[0::n_f] += fv @ np.array(fw)
        return dofs, K, f

    # -- hp level sequence (Fig. hpmultigrid) --------------------------------
    def level_sequence(self):
        """(p,k) ... (1,k), (1,k-1) ... (1,0); trailing levels without DOFs are dropped
        (when every base element is refined, no base vertex is active and (1,0) is empty)."""
        p, k = self.cfg.p, int(self.dof_depth.max()) if self.ndof else 0
        seq = [(q, k) for q in range(p, 0, -1)] + [(1, kc) for kc in range(k - 1, -1, -1)]
        while len(seq) > 1 and len(self.level_dofs(*seq[-1])) == 0:
            seq.pop()
        return seq

    def level_dofs(self, q, kc):
        return np.nonzero((self.dof_order <= q) & (self.dof_depth <= kc))[0]



class MlhpLevel:
    def __init__(self, prob, q, kc, block, omega, need_blocks=True):
        self.q, self.kc = q, kc
        self.idx = prob.level_dofs(q, kc)
        self.n = len(self.idx)
        self.A = prob.A[self.idx][:, self.idx].tocsr()
        self.omega = omega
        if not need_blocks:
            return
        pos = np.full(prob.ndof, -1, dtype=np.int64)
        pos[self.idx] = np.arange(self.n)
        M = prob.mesh
        # level DOFs nonzero on each leaf
        leaf_level = {}
        for leaf, d in zip(M.leaves, prob.leaf_dofs):
            g = pos[d]
            leaf_level[leaf] = np.unique(g[g >= 0])

        n, d = M.n, M.dim
        base_leaves = {}
        for l in M.leaves:
            base = tuple(x >> l[0] for x in l[1])
            base_leaves.setdefault(base, []).append(leaf_level[l])
        groups = []
        if block == "element":   # one block per BASE element (Fig. 7 caption, reading R26)
            for be in itertools.product(range(n), repeat=d):
                groups.append(base_leaves[be[::-1]])
        else:   # patch: the 2^d base elements around each base vertex (Fig. 7b)
            for v in itertools.product(range(n + 1), repeat=d):
                v = v[::-1]
                grp = []
                for corner in itertools.product((0, 1), repeat=d):
                    be = tuple(v[a] - 1 + corner[a] for a in range(d))
                    if all(0 <= x < n for x in be):
                        grp.extend(base_leaves[be])
                groups.append(grp)
        seen = set()
        self.blocks = []
        for grp in groups:
            if not grp:
                continue
            b = np.unique(np.concatenate(grp))
            t = tuple(b.tolist())
            if len(b) and t not in seen:
                seen.add(t)
                self.blocks.append(b)
        self.inv = [np.linalg.inv(self.A[b][:, b].toarray()) for b in self.blocks]

    def set_blocks(self, blocks, inverses):
        """Identical-setup parity protocol (as mg.Level.set_blocks): externally supplied blocks
        (level-local index arrays) and inverses replace this level's own."""
        self.blocks = [np.asarray(b, dtype=np.int64) for b in blocks]
        self.inv = [np.asarray(a, dtype=np.float64) for a in inverses]

    order_seed = None   # accumulate in a seeded random block order (rounding-spread measurement, R18/R24)
    noise = None        # (rng) rounding model of the same measurement

    def schwarz(self, r):
        """M^{-1} r = sum_i P_i A_i^{-1} P_i^T r (Eq. AdditiveSchwarz), serial order."""
        order = range(len(self.blocks))
        if self.order_seed is not None:
            order = np.random.default_rng(self.order_seed).permutation(len(self.blocks))
        idx = np.concatenate([self.blocks[i] for i in order])
        vals = np.concatenate([self.inv[i] @ r[self.blocks[i]] for i in order])
        if self.noise is not None:   # rounding model (Higham-Mary probabilistic bound): sqrt(m_i) eps |A_i^-1||r_i| N(0,1)
            mag = np.concatenate([np.sqrt(len(self.blocks[i])) * (np.abs(self.inv[i]) @ np.abs(r[self.blocks[i]]))
                                  for i in order])
            out = np.bincount(idx, weights=vals, minlength=self.n)
            return out + np.finfo(float).eps * np.bincount(idx, weights=mag, minlength=self.n) * \
                self.noise.standard_normal(self.n)
        return np.bincount(idx, weights=vals, minlength=self.n)


class MlhpHierarchy:
    """hp-multigrid (Algorithm 1, reading R1) over the hp level sequence."""

    def __init__(self, prob, block=None, omega=None, n_pre=None, n_post=None, coarse=None,
                 coarse_rtol=None, coarse_maxit=None):
        cfg = prob.cfg
        self.prob = prob
        self.block = block or cfg.block
        self.omega = omega if omega is not None else cfg.replace(block=self.block, omega=None).omega_value
        self.n_pre = cfg.n_pre if n_pre is None else n_pre
        self.n_post = cfg.n_post if n_post is None else n_post
        self.coarse = coarse or cfg.coarse
        self.coarse_rtol = cfg.coarse_rtol if coarse_rtol is None else coarse_rtol
        self.coarse_maxit = cfg.coarse_maxit if coarse_maxit is None else coarse_maxit
        self.seq = prob.level_sequence()
        self.levels = []
        for i, (q, kc) in enumerate(self.seq):
            last = i == len(self.seq) - 1
            if last:   # coarse AS is elementwise and undamped (R4, R11)
                self.levels.append(MlhpLevel(prob, q, kc, "element", 1.0, need_blocks=self.coarse == "as_pcg"))
            else:
                self.levels.append(MlhpLevel(prob, q, kc, self.block, self.omega))
        self.sel = [np.searchsorted(self.levels[i].idx, self.levels[i + 1].idx)
                    for i in range(len(self.levels) - 1)]
        c = self.levels[-1]
        if self.coarse == "direct":
            self.lu = sla.lu_factor(c.A.toarray())
        self.coarse_iters = []

    def set_coarse_inverse(self, inv):
        """Identical-setup parity protocol: apply a supplied dense inverse as the direct coarse solve."""
        self.coarse_inv = np.asarray(inv, dtype=np.float64)

    def coarse_solve(self, b):
        lv = self.levels[-1]
        if self.coarse == "direct":
            if getattr(self, "coarse_inv", None) is not None:
                return self.coarse_inv @ b
            return sla.lu_solve(self.lu, b)
        x, it = pcg(lambda v: lv.A @ v, b, lv.schwarz, self.coarse_rtol, self.coarse_maxit, rel_to="r0")
        self.coarse_iters.append(it)
        return x

    noise = None   # (rng) rounding model for spread measurements (Higham-Mary probabilistic bound:
    #               a dot product of k terms errs by ~ sqrt(k) eps sum |terms|): residuals get
    #               sqrt(nnz_row) eps |A||x| N(0,1)

    def _res(self, lv, b, x):
        r = b - lv.A @ x
        if self.noise is not None:
            k = np.sqrt(np.diff(lv.A.indptr) + 1.0)
            r = r + np.finfo(float).eps * k * (abs(lv.A) @ np.abs(x) + np.abs(b)) * self.noise.standard_normal(len(r))
        return r

    def vcycle(self, b, i=0):
        if i == len(self.levels) - 1:
            return self.coarse_solve(b)
        lv = self.levels[i]
        w = self.omega
        x = np.zeros(lv.n)
        for _ in range(self.n_pre):
            x = x + w * lv.schwarz(self._res(lv, b, x))
        r = self._res(lv, b, x)
        x[self.sel[i]] += self.vcycle(r[self.sel[i]], i + 1)
        for _ in range(self.n_post):
            x = x + w * lv.schwarz(self._res(lv, b, x))
        return x

    def mg_solve(self, b, rtol=None, maxit=None):
        """hp-multigrid as a stand-alone solver (as mg.Hierarchy.mg_solve):
        x_i = x_{i-1} + V(b - A x_{i-1}), stop at ||r_i|| / ||b|| < rtol or maxit V-cycles."""
        cfg = self.prob.cfg
        rtol = cfg.rtol if rtol is None else rtol
        maxit = cfg.maxit if maxit is None else maxit
        A = self.levels[0].A
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

    def fcg(self, b, rtol=None, maxit=None):
        cfg = self.prob.cfg
        rtol = cfg.rtol if rtol is None else rtol
        maxit = cfg.maxit if maxit is None else maxit
        A = self.levels[0].A
        return fcg(lambda v: A @ v, b, self.vcycle, rtol, maxit)

    def as_pcg(self, b, rtol, maxit):
        """CG preconditioned by the fine-level additive Schwarz alone (the paper's left tables)."""
        lv = self.levels[0]
        nb = np.linalg.norm(b)
        x, it = pcg(lambda v: lv.A @ v, b, lv.schwarz, rtol * nb / max(np.linalg.norm(b), 1e-300), maxit)
        return x, it
