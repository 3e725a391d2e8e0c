"""Multi-process CPU tests (gloo, world size 2 and 3) of the slab decomposition's HOST logic
(include/fcm_mg.h "multi-GPU"): the partition, each rank's local layout and
DOF keys, the interface planes in exchange order, the owner mask used by the dots, and the
coarse all-gather map -- the same C++ functions the library's NCCL path runs on.

Each rank applies the ORACLE's element matrices of its own cells only (element-by-element,
numpy) to a vector in its local layout, sums the interface planes with its neighbours through
gloo in the library's exchange order, and must then hold exactly the oracle's global result
restricted to its local DOFs: operator apply, residual (b counted once, by the lower rank),
elementwise additive-Schwarz update, owned dot products, and the replicated coarse vector."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _exchange(v, lo, hi, rank, world):
    """Sum interface planes with the neighbours (gloo), in the library's order."""
    mine = {"lo": v[lo].copy(), "hi": v[hi].copy()}
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    out = v.copy()
    if len(lo):
        out[lo] += allp[rank - 1]["hi"]
    if len(hi):
        out[hi] += allp[rank + 1]["lo"]
    return out


def _cell_matrix(P, c):
    kind = P.kinds[c]
    if kind == 2:
        return P.cut_K[P.cut_index[c]]
    return P.K_ref * (P.cfg.alpha if kind == 1 else 1.0)


def _worker(rank, world, port, cfg_args, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.mg import Hierarchy
        from oracle.problem import Problem
        from paper_2010_00881_b200.fcm import slab_bounds, slab_coarse_map, slab_layout
        from workloads import small_config

        cfg = small_config(**cfg_args)
        P = Problem(cfg)
        n, dim, p = cfg.n, cfg.dim, cfg.p
        z0, z1 = slab_bounds(n, world, rank)
        plane = n ** (dim - 1)
        owned_cells = np.arange(z0 * plane, z1 * plane)
        rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)  # noqa: E731
        rng = np.random.default_rng(7)
        x = rng.standard_normal(P.dof.ndof)
        out = {}
        for q in (p, 1):
            keys, own, lo, hi = slab_layout(cfg, z0, z1, q)
            pos = np.searchsorted(P.dof.keys, keys)
            assert np.array_equal(P.dof.keys[pos], keys), "local keys are global DOF keys"
            Iq = P.dof.level_dofs(q)
            xq = np.zeros_like(x)
            xq[Iq] = x[Iq]
            Aq = P.A[Iq][:, Iq]
            mq = P.dof.level_m(q)
            # operator apply over the owned cells only, then the interface exchange
            yp = np.zeros(P.dof.ndof)
            for c in owned_cells:
                idx = P.dof.cell_dofs[c, :mq]
                ok = idx >= 0
                K = _cell_matrix(P, c)[:mq, :mq]
                yp[idx[ok]] += K[np.ix_(ok, ok)] @ xq[idx[ok]]
            y = _exchange(yp[pos], lo, hi, rank, world)
            ref = np.zeros_like(x)
            ref[Iq] = Aq @ x[Iq]
            out[f"apply_q{q}"] = rel(y, ref[pos])
            # owned dot product, summed over ranks
            d = torch.tensor([float(np.dot(xq[pos][own], y[own]))], dtype=torch.float64)
            dist.all_reduce(d)
            out[f"dot_q{q}"] = abs(d.item() - float(xq[Iq] @ ref[Iq])) / abs(float(xq[Iq] @ ref[Iq]))
            # residual: b counted by the lower rank only (bottom plane zeroed on this rank)
            bq = np.zeros_like(x)
            bq[Iq] = P.b[Iq]
            r0 = bq[pos].copy()
            r0[lo] = 0.0
            r = _exchange(r0 - yp[pos], lo, hi, rank, world)
            out[f"residual_q{q}"] = rel(r, (bq - ref)[pos])
        # additive-Schwarz update of level p: blocks of the owned cells only, then exchange
        H = Hierarchy(P)
        lv = H.levels[p]
        keys, own, lo, hi = slab_layout(cfg, z0, z1, p)
        pos = np.searchsorted(P.dof.keys, keys)
        lpos = np.full(P.dof.ndof, -1)
        lpos[lv.idx] = np.arange(lv.n)
        rl = rng.standard_normal(lv.n)
        bi = 0
        dp = np.zeros(lv.n)
        mq = P.dof.level_m(p)
        for c in range(n ** dim):
            g = P.dof.cell_dofs[c, :mq]
            if not np.any(g >= 0):
                continue
            blk = lv.blocks[bi]
            if z0 * plane <= c < z1 * plane:
                dp[blk] += lv.omega * (lv.inv[bi] @ rl[blk])
            bi += 1
        full = np.zeros(P.dof.ndof)
        full[lv.idx] = dp
        d_loc = _exchange(full[pos], lo, hi, rank, world)
        ref = np.zeros(P.dof.ndof)
        ref[lv.idx] = lv.omega * lv.schwarz(rl)
        out["smoother"] = rel(d_loc, ref[pos])
        # replicated coarse level: local level-1 slots <-> global (class-major) level-1 slots
        gm = slab_coarse_map(cfg, z0, z1)
        k1, own1, _, _ = slab_layout(cfg, z0, z1, 1)
        kg, _, _, _ = slab_layout(cfg, 0, n, 1)
        out["coarse_keys_match"] = bool(np.array_equal(kg[gm], k1))
        owned_g = [None] * world
        dist.all_gather_object(owned_g, gm[own1])
        allg = np.sort(np.concatenate(owned_g))
        out["coarse_owned_is_partition"] = bool(np.array_equal(allg, np.arange(len(kg))))
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg_args", [
    dict(dim=3, n=5, p=2, voids=2, seed=5),
    dict(dim=3, n=4, p=3, space="trunk", physics="elasticity", voids=1, seed=6),
    dict(dim=2, n=7, p=3, voids=1, seed=2),
])
def test_slab_host_logic_matches_oracle(world, cfg_args):
    if cfg_args["n"] < world:
        pytest.skip("fewer layers than ranks")
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), cfg_args, results), nprocs=world, join=True)
    assert len(results) == world
    for rank, out in results.items():
        for k, v in out.items():
            if isinstance(v, bool):
                assert v, (rank, k)
            else:
                assert v <= 1e-12, (rank, k, v)


def test_slab_bounds_partition():
    from paper_2010_00881_b200.fcm import slab_bounds
    for n in (1, 5, 32, 257):
        for world in (1, 2, 3, 8):
            if world > n:
                continue
            b = [slab_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
            sizes = [z1 - z0 for z0, z1 in b]
            assert max(sizes) - min(sizes) <= 1


def _allreduce_np(v):
    t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _dist_gmg_worker(rank, world, port, cfg_args, results):
    """The DISTRIBUTED h-coarsened coarse solve (library: coarse_dist / gmg_vcycle_dist; P:227
    Remark) emulated with numpy on each rank's slab: the p=1 level stays slab partitioned (its
    operator and its h-level-0 elementwise AS sweeps over the owned cells + interface exchange,
    owned dots all-reduced), the restriction to h-level 1 is each slab's OWNED rows of P^T r
    all-reduced, the h-levels below run replicated, the prolongation is the slab's rows of P e.
    Must reproduce the oracle's global CG + geometric V-cycle (GeometricLevels)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.mg import Hierarchy
        from oracle.problem import Problem
        from paper_2010_00881_b200.fcm import slab_bounds, slab_layout
        from workloads import small_config

        cfg = small_config(**cfg_args, coarse="gmg_pcg")
        P = Problem(cfg)
        H = Hierarchy(P)
        G = H.gmg
        lv = H.levels[1]
        n, dim = cfg.n, cfg.dim
        z0, z1 = slab_bounds(n, world, rank)
        plane = n ** (dim - 1)
        keys, own, lo, hi = slab_layout(cfg, z0, z1, 1)
        gpos = np.searchsorted(P.dof.keys, keys)          # global DOF of each local slot
        lpos = np.full(P.dof.ndof, -1)
        lpos[lv.idx] = np.arange(lv.n)
        l1 = lpos[gpos]                                    # level-1 (oracle order) position of each local slot
        assert np.all(l1 >= 0)
        m1 = P.dof.level_m(1)
        owned_cells = set(range(z0 * plane, z1 * plane))
        # local operator / smoother over the owned cells, then the interface exchange
        cell_blocks = []
        bi = 0
        for c in range(n ** dim):
            g = P.dof.cell_dofs[c, :m1]
            if not np.any(g >= 0):
                continue
            if c in owned_cells:
                cell_blocks.append((c, lv.blocks[bi], lv.inv[bi]))
            bi += 1
        inv_l1 = np.full(lv.n, -1)
        inv_l1[l1] = np.arange(len(l1))

        def apply(v):
            y = np.zeros(lv.n)
            vg = np.zeros(lv.n)
            vg[l1] = v
            for c, _, _ in cell_blocks:
                idx = P.dof.cell_dofs[c, :m1]
                ok = idx >= 0
                K = _cell_matrix(P, c)[:m1, :m1]
                rows = lpos[idx[ok]]
                y[rows] += K[np.ix_(ok, ok)] @ vg[rows]
            return _exchange(y[l1], lo, hi, rank, world)

        def smooth(r, w):
            d = np.zeros(lv.n)
            rg = np.zeros(lv.n)
            rg[l1] = r
            for _, blk, inv in cell_blocks:
                d[blk] += w * (inv @ rg[blk])
            return _exchange(d[l1], lo, hi, rank, world)

        def dot(a, b):
            return float(_allreduce_np(np.array([np.dot(a[own], b[own])]))[0])

        def vcycle_dist(b):
            w = G.omega
            x = np.zeros_like(b)
            for _ in range(G.n_pre):
                x = x + smooth(b - apply(x), w)
            r = b - apply(x)
            full = np.zeros(lv.n)
            full[l1[own]] = r[own]                         # this slab's owned rows only
            bc = _allreduce_np(G.P[0].T @ full)            # all-reduced restriction
            ec = G.vcycle(bc, 1)                           # replicated h-levels
            x = x + (G.P[0] @ ec)[l1]
            for _ in range(G.n_post):
                x = x + smooth(b - apply(x), w)
            return x

        # right-hand side: the level-1 part of the load
        b_glob = P.b[lv.idx]
        ref = H.coarse_solve(b_glob)
        it_ref = H.coarse_iters[-1]
        b = b_glob[l1]
        x = np.zeros_like(b)
        r = b.copy()
        z = vcycle_dist(r)
        rz, rr0 = dot(r, z), dot(r, r)
        p = z.copy()
        it = 0
        while True:
            q = apply(p)
            a = rz / dot(p, q)
            x += a * p
            r -= a * q
            it += 1
            if dot(r, r) < H.coarse_rtol ** 2 * rr0 or it >= H.coarse_maxit:
                break
            z = vcycle_dist(r)
            rzn = dot(r, z)
            p = z + (rzn / rz) * p
            rz = rzn
        rel = np.linalg.norm(x - ref[l1]) / np.linalg.norm(ref[l1])
        results[rank] = {"rel": float(rel), "it": it, "it_ref": int(it_ref)}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg_args", [
    dict(dim=3, n=8, p=2, voids=2, seed=5),
    dict(dim=2, n=16, p=3, voids=1, seed=2),
    dict(dim=3, n=8, p=2, physics="elasticity", voids=1, seed=6),
])
def test_distributed_gmg_coarse_matches_oracle(world, cfg_args):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_dist_gmg_worker, args=(world, _free_port(), cfg_args, results), nprocs=world, join=True)
    assert len(results) == world
    for rank, out in results.items():
        assert abs(out["it"] - out["it_ref"]) <= 1, (rank, out)
        assert out["rel"] <= 1e-9, (rank, out)
