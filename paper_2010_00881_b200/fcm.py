"""Thin Python API over the C ABI (argument marshalling only; every step of the hot path
runs in the sm_100a kernels of libfcm_mg.so).  PyTorch supplies device memory and streams.

    prob = generate(cfg)                      # workload generator (C++, setup)
    solver = Solver.from_problem(cfg, prob)   # fcm_mg_setup
    b = solver.load(prob)                     # fcm_mg_load
    x, iters, hist = solver.pcg_solve(b)      # fcm_pcg_solve (flexible CG + V-cycle)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import Grid, HpSpec, Params, Physics, Slab, check

COARSE = {"direct": 0, "as_pcg": 1, "jacobi_pcg": 2, "gmg_pcg": 3}
BLOCK = {"element": 0, "patch": 1}


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _vecptr(t, n, device=None, name="vector"):
    """Pointer of a caller-supplied vector after checking what the C ABI assumes (fp64,
    contiguous, exactly n entries, on the handle's device -- or on the host when device is
    None); a mismatch raises ValueError instead of reading or writing out of bounds."""
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if t.dtype != torch.float64:
        raise ValueError(f"{name}: dtype {t.dtype}, expected torch.float64")
    if not t.is_contiguous():
        raise ValueError(f"{name}: not contiguous")
    if t.numel() != n:
        raise ValueError(f"{name}: {t.numel()} entries, expected {n}")
    if device is None:
        if t.is_cuda:
            raise ValueError(f"{name}: expected a host tensor")
    elif t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device}")
    return C.c_void_p(t.data_ptr())


def grid_of(cfg) -> Grid:
    g = Grid()
    g.dim = cfg.dim
    g.n[0] = cfg.n
    g.n[1] = cfg.n
    g.n[2] = cfg.n if cfg.dim == 3 else 1
    g.h = 1.0 / cfg.n
    g.p = cfg.p
    g.space = 0 if cfg.space == "tensor" else 1
    g.n_f = cfg.n_f
    g.dirichlet_faces = cfg.dirichlet_mask
    return g


def physics_of(cfg) -> Physics:
    ph = Physics()
    ph.kind = 0 if cfg.physics == "poisson" else 1
    ph.alpha = cfg.alpha
    ph.E = cfg.E
    ph.nu = cfg.nu
    ph.depth = cfg.depth
    ph.traction_face = cfg.traction_face
    return ph


def params_of(cfg, stream=None, **over) -> Params:
    pr = Params()
    pr.block = BLOCK[over.get("block", cfg.block)]
    om = over.get("omega")
    if om is None:
        om = cfg.omega if cfg.omega is not None else cfg.replace(block=over.get("block", cfg.block)).omega_value
    pr.omega = om
    pr.n_pre = over.get("n_pre", cfg.n_pre)
    pr.n_post = over.get("n_post", cfg.n_post)
    pr.coarse = COARSE[over.get("coarse", cfg.coarse)]
    pr.coarse_rtol = over.get("coarse_rtol", cfg.coarse_rtol)
    pr.coarse_maxit = over.get("coarse_maxit", cfg.coarse_maxit)
    if stream is None:
        stream = torch.cuda.current_stream().cuda_stream
    pr.stream = stream
    return pr


def element_size(cfg) -> int:
    g = grid_of(cfg)
    m = _lib.lib().fcm_element_size(C.byref(g))
    check(min(m, 0))
    return m


@dataclass
class GenProblem:
    kind: np.ndarray        # uint8 [ncell]
    cut_cells: np.ndarray   # int64 [n_cut]
    K_ref: np.ndarray       # [m, m]
    f_ref: np.ndarray       # [m]
    cut_K: np.ndarray       # [n_cut, m, m]
    cut_f: np.ndarray       # [n_cut, m]
    f_traction: np.ndarray  # [m]


def classify(cfg, centres, radii):
    centres = np.ascontiguousarray(centres, dtype=np.float64)
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    g = grid_of(cfg)
    kind = np.zeros(cfg.n ** cfg.dim, dtype=np.uint8)
    ncut = C.c_int64(0)
    check(_lib.lib().fcm_gen_classify(C.byref(g), len(radii), _ptr(centres), _ptr(radii), _ptr(kind),
                                      C.byref(ncut)))
    return kind, ncut.value


def device_quadrature_ok(cfg) -> bool:
    """fcm_gen_cut_matrices_device handles this workload (Poisson, depth <= 4, m <= 128) and a
    CUDA device is present."""
    return (cfg.physics == "poisson" and cfg.depth <= 4 and (cfg.p + 1) ** cfg.dim <= 128
            and torch.cuda.is_available())


def generate(cfg, centres=None, radii=None, threads: int = 0, cut_cells=None, kind=None,
             device=None) -> GenProblem:
    """Workload generator (fcm_gen_classify + fcm_gen_element_matrices).  cut_cells: restrict
    the cut-cell quadrature to these cells (slab + ghost layers in multi-GPU runs).
    device: cut-cell quadrature on the GPU (fcm_gen_cut_matrices_device); None = whenever
    device_quadrature_ok(cfg)."""
    from workloads import config_voids
    if centres is None:
        centres, radii = config_voids(cfg)
    centres = np.ascontiguousarray(centres, dtype=np.float64)
    radii = np.ascontiguousarray(radii, dtype=np.float64)
    L = _lib.lib()
    g = grid_of(cfg)
    ph = physics_of(cfg)
    if kind is None:
        kind, _ = classify(cfg, centres, radii)
    if cut_cells is None:
        cut_cells = np.nonzero(kind == 2)[0].astype(np.int64)
    cut_cells = np.ascontiguousarray(cut_cells, dtype=np.int64)
    m = element_size(cfg)
    K_ref = np.zeros((m, m))
    f_ref = np.zeros(m)
    cut_K = np.zeros((len(cut_cells), m, m))
    cut_f = np.zeros((len(cut_cells), m))
    f_tr = np.zeros(m)
    if device is None:
        device = device_quadrature_ok(cfg)
    if device:
        # K_ref, f_ref, f_traction on the host (one cell), the cut cells on the device
        check(L.fcm_gen_element_matrices(C.byref(g), C.byref(ph), len(radii), _ptr(centres), _ptr(radii),
                                         _ptr(K_ref), _ptr(f_ref), 0, None, None, None, _ptr(f_tr), threads))
        torch.cuda.init()
        check(L.fcm_gen_cut_matrices_device(C.byref(g), C.byref(ph), len(radii), _ptr(centres), _ptr(radii),
                                            len(cut_cells), _ptr(cut_cells), _ptr(cut_K), _ptr(cut_f)))
    else:
        check(L.fcm_gen_element_matrices(C.byref(g), C.byref(ph), len(radii), _ptr(centres), _ptr(radii),
                                         _ptr(K_ref), _ptr(f_ref), len(cut_cells), _ptr(cut_cells),
                                         _ptr(cut_K), _ptr(cut_f), _ptr(f_tr), threads))
    return GenProblem(kind, cut_cells, K_ref, f_ref, cut_K, cut_f, f_tr)


# ---- slab decomposition (multi-GPU; include/fcm_mg.h "multi-GPU") -----------------------
def slab_bounds(n: int, nranks: int, rank: int):
    a, b = C.c_int32(), C.c_int32()
    check(_lib.lib().fcm_slab_bounds(n, nranks, rank, C.byref(a), C.byref(b)))
    return a.value, b.value


def slab_layout(cfg, z_begin: int, z_end: int, q: int):
    """Host-only local layout of a slab: (keys, owned mask, bottom plane slots, top plane slots)."""
    L = _lib.lib()
    g = grid_of(cfg)
    n, nlo, nhi = C.c_int64(), C.c_int64(), C.c_int64()
    check(L.fcm_slab_layout(C.byref(g), z_begin, z_end, q, C.byref(n), None, None, C.byref(nlo), None,
                            C.byref(nhi), None))
    keys = np.zeros(n.value, dtype=np.int64)
    own = np.zeros(n.value, dtype=np.uint8)
    lo = np.zeros(nlo.value, dtype=np.int32)
    hi = np.zeros(nhi.value, dtype=np.int32)
    check(L.fcm_slab_layout(C.byref(g), z_begin, z_end, q, C.byref(n), _ptr(keys), _ptr(own), C.byref(nlo),
                            _ptr(lo) if len(lo) else None, C.byref(nhi), _ptr(hi) if len(hi) else None))
    return keys, own.astype(bool), lo, hi


def slab_coarse_map(cfg, z_begin: int, z_end: int) -> np.ndarray:
    L = _lib.lib()
    g = grid_of(cfg)
    n = C.c_int64()
    check(L.fcm_slab_coarse_map(C.byref(g), z_begin, z_end, C.byref(n), None))
    out = np.zeros(n.value, dtype=np.int64)
    check(L.fcm_slab_coarse_map(C.byref(g), z_begin, z_end, C.byref(n), _ptr(out)))
    return out


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    check(_lib.lib().fcm_nccl_unique_id(buf))
    return bytes(buf)


class Solver:
    """Owns an fcm_mg handle (device hierarchy, Schwarz inverses, graphs)."""

    def __init__(self, cfg, K_ref, cell_kind, cut_cells, cut_K, alpha=None, stream=None, slab=None,
                 coarse_cut=None, **over):
        self.cfg = cfg
        L = _lib.lib()
        self._g = grid_of(cfg)
        self._p = params_of(cfg, stream, **over)
        K_ref = np.ascontiguousarray(K_ref, dtype=np.float64)
        cell_kind = np.ascontiguousarray(cell_kind, dtype=np.uint8)
        cut_cells = np.ascontiguousarray(cut_cells, dtype=np.int64)
        cut_K = np.ascontiguousarray(cut_K, dtype=np.float64)
        h = C.c_void_p()
        a = cfg.alpha if alpha is None else alpha
        if slab is None:
            check(L.fcm_mg_setup(C.byref(self._g), C.byref(self._p), _ptr(K_ref), _ptr(cell_kind), a,
                                 len(cut_cells), _ptr(cut_cells), _ptr(cut_K), C.byref(h)))
        else:
            rank, nranks, z0, z1, nccl_id = slab
            self._idbuf = C.create_string_buffer(bytes(nccl_id) if nccl_id else b"\0" * 128, 128)
            sl = Slab(rank, nranks, z0, z1, C.cast(self._idbuf, C.c_void_p))
            cc, cK1 = coarse_cut if coarse_cut is not None else (np.zeros(0, np.int64), np.zeros(0))
            cc = np.ascontiguousarray(cc, dtype=np.int64)
            cK1 = np.ascontiguousarray(cK1, dtype=np.float64)
            check(L.fcm_mg_setup_slab(C.byref(self._g), C.byref(self._p), C.byref(sl), _ptr(K_ref),
                                      _ptr(cell_kind), a, len(cut_cells), _ptr(cut_cells), _ptr(cut_K),
                                      len(cc), _ptr(cc), _ptr(cK1), C.byref(h)))
        self.slab = slab
        self._h = h
        self.device = torch.device("cuda", torch.cuda.current_device())

    @classmethod
    def distributed(cls, cfg, rank: int, nranks: int, threads: int = 0, **over):
        """Slab-decomposed solver over torch.distributed ranks (one GPU each).  Each rank runs
        the generator for its owned + ghost cell layers; the leading p = 1 blocks of every cut
        cell (replicated coarse level) and the NCCL id are exchanged through torch.distributed
        (plumbing).  Returns (solver, local GenProblem restricted to the slab)."""
        import torch.distributed as dist
        from workloads import config_voids
        n = cfg.n
        z0, z1 = slab_bounds(n, nranks, rank)
        centres, radii = config_voids(cfg)
        kind, _ = classify(cfg, centres, radii)
        plane = n ** (cfg.dim - 1)
        lo, hi = max(z0 - 1, 0) * plane, min(z1 + 1, n) * plane
        cut_all = np.nonzero(kind == 2)[0].astype(np.int64)
        cut_ext = cut_all[(cut_all >= lo) & (cut_all < hi)]
        G = generate(cfg, centres, radii, threads=threads, cut_cells=cut_ext, kind=kind)
        m1 = (2 ** cfg.dim) * cfg.n_f
        own = (cut_ext >= z0 * plane) & (cut_ext < z1 * plane)
        mine = (cut_ext[own], np.ascontiguousarray(G.cut_K[own][:, :m1, :m1]))
        parts = [None] * nranks
        dist.all_gather_object(parts, mine)
        cc = np.concatenate([p_[0] for p_ in parts]) if parts else np.zeros(0, np.int64)
        cK1 = np.concatenate([p_[1] for p_ in parts]) if parts else np.zeros((0, m1, m1))
        order = np.argsort(cc)
        ids = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        S = cls(cfg, G.K_ref, kind, cut_ext, G.cut_K, slab=(rank, nranks, z0, z1, ids[0]),
                coarse_cut=(cc[order], cK1[order]), **over)
        return S, G

    @classmethod
    def from_problem(cls, cfg, prob: GenProblem, **over):
        return cls(cfg, prob.K_ref, prob.kind, prob.cut_cells, prob.cut_K, **over)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().fcm_mg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- queries --------------------------------------------------------------------------
    def ndofs(self, q=None) -> int:
        q = self.cfg.p if q is None else q
        n = C.c_int64()
        check(_lib.lib().fcm_mg_ndofs(self._h, q, C.byref(n)))
        return n.value

    def level_m(self, q) -> int:
        m = C.c_int32()
        check(_lib.lib().fcm_mg_level_m(self._h, q, C.byref(m)))
        return m.value

    def irregular_blocks(self, q) -> int:
        n, t = C.c_int64(), C.c_int32()
        check(_lib.lib().fcm_mg_block_counts(self._h, q, C.byref(n), C.byref(t)))
        return n.value

    def block_size(self, q) -> int:
        """m_b of level q's Schwarz blocks (element size, or (2q+1)^d patch slots)."""
        n, mb = C.c_int64(), C.c_int32()
        check(_lib.lib().fcm_mg_export_block_inverses(self._h, q, C.byref(n), C.byref(mb), None, None, None))
        return mb.value

    def block_counts(self, q):
        n, t = C.c_int64(), C.c_int32()
        check(_lib.lib().fcm_mg_block_counts(self._h, q, C.byref(n), C.byref(t)))
        return n.value, t.value

    def lowrank_info(self, q):
        """(number of low-rank individual patches, total entries of their C matrices) on level q."""
        a, b = C.c_int64(), C.c_int64()
        check(_lib.lib().fcm_mg_lowrank_info(self._h, q, C.byref(a), C.byref(b)))
        return a.value, b.value

    def export_block_inverses(self, q):
        """(anchors [n], dof_index [n, m_b] (-1: no free DOF), inverses [n, m_b, m_b]) of level
        q's Schwarz blocks exactly as the smoother applies them (fcm_mg_export_block_inverses,
        the parity protocol of SURVEY §8(c))."""
        L = _lib.lib()
        n, mb = C.c_int64(), C.c_int32()
        check(L.fcm_mg_export_block_inverses(self._h, q, C.byref(n), C.byref(mb), None, None, None))
        anchors = np.zeros(n.value, dtype=np.int64)
        idx = np.zeros((n.value, mb.value), dtype=np.int32)
        inv = np.zeros((n.value, mb.value, mb.value))
        check(L.fcm_mg_export_block_inverses(self._h, q, C.byref(n), C.byref(mb), _ptr(anchors),
                                             _ptr(idx), _ptr(inv)))
        return anchors, idx, inv

    def dof_keys(self) -> np.ndarray:
        k = np.zeros(self.ndofs(), dtype=np.int64)
        check(_lib.lib().fcm_mg_dof_keys(self._h, _ptr(k)))
        return k

    def launches(self) -> int:
        v = C.c_int64()
        check(_lib.lib().fcm_mg_launch_count(self._h, C.byref(v)))
        return v.value

    def coarse_info(self):
        """(kernel name, cooperative CTAs, brick size) of the coarse solver (fcm_mg_coarse_info)."""
        k, nb = C.c_int32(), C.c_int32()
        t = (C.c_int32 * 3)()
        check(_lib.lib().fcm_mg_coarse_info(self._h, C.byref(k), C.byref(nb), t))
        name = {0: "k_dense_gemv", 1: "k_coarse_pcg", 2: "k_coarse_tiled", 3: "gmg_pcg"}[k.value]
        return name, nb.value, tuple(t)

    def stats(self):
        a, b = C.c_int64(), C.c_int64()
        check(_lib.lib().fcm_mg_stats(self._h, C.byref(a), C.byref(b)))
        return {"coarse_iters": a.value, "vcycles": b.value}

    def _dv(self, t, q, name):
        return _vecptr(t, self.ndofs(q), self.device, name)

    def _vec(self, q=None):
        return torch.zeros(self.ndofs(q), dtype=torch.float64, device=self.device)

    # -- operations -------------------------------------------------------------------------
    def load(self, prob: GenProblem) -> torch.Tensor:
        b = self._vec()
        tr = prob.f_traction if self.cfg.traction_face >= 0 else None
        check(_lib.lib().fcm_mg_load(self._h, _ptr(np.ascontiguousarray(prob.f_ref)),
                                     _ptr(np.ascontiguousarray(prob.cut_f)) if len(prob.cut_f) else None,
                                     _ptr(tr), self.cfg.traction_face, _ptr(b)))
        return b

    def apply(self, x: torch.Tensor, q=None) -> torch.Tensor:
        q = self.cfg.p if q is None else q
        y = self._vec(q)
        check(_lib.lib().fcm_apply(self._h, q, self._dv(x, q, "x"), _ptr(y)))
        return y

    def smooth(self, r: torch.Tensor, x: torch.Tensor, q=None) -> torch.Tensor:
        q = self.cfg.p if q is None else q
        check(_lib.lib().fcm_mg_smooth(self._h, q, self._dv(r, q, "r"), self._dv(x, q, "x")))
        return x

    def smooth_part(self, r: torch.Tensor, x: torch.Tensor, q, part: int) -> torch.Tensor:
        """x += omega M^-1 r restricted to one block population of a patch level
        (fcm_mg_smooth_part: 1 individual patches, 2 shared-type patches, 0 both)."""
        check(_lib.lib().fcm_mg_smooth_part(self._h, q, part, self._dv(r, q, "r"), self._dv(x, q, "x")))
        return x

    def coarse_solve(self, r: torch.Tensor):
        x = self._vec(1)
        it = C.c_int32()
        check(_lib.lib().fcm_mg_coarse_solve(self._h, self._dv(r, 1, "r"), _ptr(x), C.byref(it)))
        return x, it.value

    def vcycle(self, r: torch.Tensor) -> torch.Tensor:
        z = self._vec()
        check(_lib.lib().fcm_mg_vcycle(self._h, self._dv(r, None, "r"), _ptr(z)))
        return z

    def pcg_solve(self, b: torch.Tensor, rtol=None, maxit=None, x=None):
        rtol = self.cfg.rtol if rtol is None else rtol
        maxit = self.cfg.maxit if maxit is None else maxit
        x = self._vec() if x is None else x
        it = C.c_int32()
        hist = np.zeros(maxit + 1)
        rc = _lib.lib().fcm_pcg_solve(self._h, self._dv(b, None, "b"), self._dv(x, None, "x"), rtol, maxit,
                                      C.byref(it), _ptr(hist))
        check(rc, allow_not_converged=True)
        return x, it.value, hist[: it.value + 1]

    def mg_solve(self, b: torch.Tensor, rtol=None, maxit=None, x=None):
        """Stand-alone multigrid x_i = x_{i-1} + V(b - A x_{i-1}) (fcm_mg_solve)."""
        rtol = self.cfg.rtol if rtol is None else rtol
        maxit = self.cfg.maxit if maxit is None else maxit
        x = self._vec() if x is None else x
        it = C.c_int32()
        hist = np.zeros(maxit + 1)
        rc = _lib.lib().fcm_mg_solve(self._h, self._dv(b, None, "b"), self._dv(x, None, "x"), rtol, maxit,
                                     C.byref(it), _ptr(hist))
        check(rc, allow_not_converged=True)
        return x, it.value, hist[: it.value + 1]

    def pcg_solve_host(self, b_host: torch.Tensor, x_host: torch.Tensor, rtol=None, maxit=None):
        rtol = self.cfg.rtol if rtol is None else rtol
        maxit = self.cfg.maxit if maxit is None else maxit
        it = C.c_int32()
        n = self.ndofs()
        rc = _lib.lib().fcm_pcg_solve_host(self._h, _vecptr(b_host, n, None, "b_host"),
                                           _vecptr(x_host, n, None, "x_host"), rtol, maxit,
                                           C.byref(it), None)
        check(rc, allow_not_converged=True)
        return it.value


# ---- multi-level hp-refinement (include/fcm_mg.h "multi-level hp") -------------
class HpDisc:
    """Host discretisation from the native generator (fcm_hp_generate): refinement trees, active
    DOFs with (depth, entity, degrees, component) keys, leaf matrices and load."""

    def __init__(self, cfg, centres=None, radii=None):
        from workloads import config_voids
        if centres is None:
            centres, radii = config_voids(cfg)
        self.cfg = cfg
        c = np.ascontiguousarray(np.asarray(centres, dtype=np.float64).reshape(-1))
        r = np.ascontiguousarray(np.asarray(radii, dtype=np.float64).reshape(-1))
        sp = HpSpec()
        sp.dim, sp.n, sp.p, sp.kmax = cfg.dim, cfg.n, cfg.p, cfg.kmax
        sp.refine = {"cut": 0, "all": 1}[cfg.refine]
        sp.dirichlet_faces = cfg.dirichlet_mask
        sp.phys = physics_of(cfg)
        sp.n_voids = len(r)
        sp.centres = c.ctypes.data_as(C.c_void_p) if len(r) else None
        sp.radii = r.ctypes.data_as(C.c_void_p) if len(r) else None
        h = C.c_void_p()
        check(_lib.lib().fcm_hp_generate(C.byref(sp), C.byref(h)))
        self._h = h
        nd, nl, nleaf, ne, nk = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
        check(_lib.lib().fcm_hp_disc_info(h, C.byref(nd), C.byref(nl), C.byref(nleaf), C.byref(ne), C.byref(nk)))
        self.ndof, self.nlevels, self.nleaves = nd.value, nl.value, nleaf.value
        self.leaf_entries, self.leaf_matrix_entries = ne.value, nk.value
        self.level_n = np.zeros(self.nlevels, np.int64)
        self.level_q = np.zeros(self.nlevels, np.int32)
        self.level_k = np.zeros(self.nlevels, np.int32)
        check(_lib.lib().fcm_hp_disc_levels(h, _ptr(self.level_n), _ptr(self.level_q), _ptr(self.level_k)))

    def keys(self) -> np.ndarray:
        k = np.zeros((self.ndof, 8), np.int32)
        check(_lib.lib().fcm_hp_disc_keys(self._h, _ptr(k)))
        return k

    def load(self) -> np.ndarray:
        b = np.zeros(self.ndof)
        check(_lib.lib().fcm_hp_disc_load(self._h, _ptr(b)))
        return b

    def leaves(self):
        ptr = np.zeros(self.nleaves + 1, np.int64)
        dofs = np.zeros(self.leaf_entries, np.int32)
        K = np.zeros(self.leaf_matrix_entries)
        info = np.zeros((self.nleaves, 5), np.int32)
        check(_lib.lib().fcm_hp_disc_leaves(self._h, _ptr(ptr), _ptr(dofs), _ptr(K), _ptr(info)))
        return ptr, dofs, K, info

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().fcm_hp_disc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HpSolver:
    """Owns an fcm_hp handle: the hp-multigrid over levels (p,k) ... (1,k) ... (1,0) on the device."""

    def __init__(self, disc: HpDisc, stream=None, **over):
        cfg = disc.cfg
        self.cfg = cfg
        self.level_n = disc.level_n.copy()
        self.nlevels = disc.nlevels
        self._p = params_of(cfg, stream, **over)
        h = C.c_void_p()
        check(_lib.lib().fcm_hp_setup(disc._h, C.byref(self._p), C.byref(h)))
        self._h = h
        self.device = torch.device("cuda", torch.cuda.current_device())

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().fcm_hp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def ndofs(self, level=0) -> int:
        return int(self.level_n[level])

    def _dv(self, t, level, name):
        return _vecptr(t, self.ndofs(level), self.device, name)

    def _vec(self, level=0):
        return torch.zeros(self.ndofs(level), dtype=torch.float64, device=self.device)

    def apply(self, x, level=0):
        y = self._vec(level)
        check(_lib.lib().fcm_hp_apply(self._h, level, self._dv(x, level, "x"), _ptr(y)))
        return y

    def smooth(self, r, x, level=0):
        check(_lib.lib().fcm_hp_smooth(self._h, level, self._dv(r, level, "r"), self._dv(x, level, "x")))
        return x

    def vcycle(self, r):
        z = self._vec()
        check(_lib.lib().fcm_hp_vcycle(self._h, self._dv(r, 0, "r"), _ptr(z)))
        return z

    def time_smooth(self, r, x, level=0, reps=20) -> float:
        """Mean ms per smoother sweep of `level` over `reps` back-to-back sweeps (events on the
        library's stream)."""
        ms = C.c_float()
        check(_lib.lib().fcm_hp_time_smooth(self._h, level, self._dv(r, level, "r"), self._dv(x, level, "x"), reps,
                                            C.byref(ms)))
        return ms.value

    def pcg_solve(self, b, rtol=None, maxit=None, x=None):
        rtol = self.cfg.rtol if rtol is None else rtol
        maxit = self.cfg.maxit if maxit is None else maxit
        x = self._vec() if x is None else x
        it = C.c_int32()
        hist = np.zeros(maxit + 1)
        rc = _lib.lib().fcm_hp_pcg_solve(self._h, self._dv(b, 0, "b"), self._dv(x, 0, "x"), rtol, maxit,
                                         C.byref(it), _ptr(hist))
        check(rc, allow_not_converged=True)
        return x, it.value, hist[: it.value + 1]

    def mg_solve(self, b, rtol=None, maxit=None, x=None):
        """Stand-alone hp-multigrid x_i = x_{i-1} + V(b - A x_{i-1}) (fcm_hp_mg_solve)."""
        rtol = self.cfg.rtol if rtol is None else rtol
        maxit = self.cfg.maxit if maxit is None else maxit
        x = self._vec() if x is None else x
        it = C.c_int32()
        hist = np.zeros(maxit + 1)
        rc = _lib.lib().fcm_hp_mg_solve(self._h, self._dv(b, 0, "b"), self._dv(x, 0, "x"), rtol, maxit,
                                        C.byref(it), _ptr(hist))
        check(rc, allow_not_converged=True)
        return x, it.value, hist[: it.value + 1]

    def export_blocks(self, level):
        """(blocks as lists of level indices, inverses) of level `level` (identical-setup parity)."""
        nb, nd, ni = C.c_int64(), C.c_int64(), C.c_int64()
        L = _lib.lib()
        check(L.fcm_hp_export_blocks(self._h, level, C.byref(nb), C.byref(nd), C.byref(ni), None, None, None))
        ptr = np.zeros(nb.value + 1, np.int64)
        dofs = np.zeros(nd.value, np.int32)
        inv = np.zeros(ni.value)
        check(L.fcm_hp_export_blocks(self._h, level, C.byref(nb), C.byref(nd), C.byref(ni), _ptr(ptr), _ptr(dofs),
                                     _ptr(inv)))
        blocks, invs, o = [], [], 0
        for i in range(nb.value):
            d = dofs[ptr[i]:ptr[i + 1]].astype(np.int64)
            m = len(d)
            blocks.append(d)
            invs.append(inv[o:o + m * m].reshape(m, m))
            o += m * m
        return blocks, invs

    def stats(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        check(_lib.lib().fcm_hp_stats(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return {"launches": a.value, "coarse_iters": b.value, "vcycles": c.value}
