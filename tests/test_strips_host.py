"""CPU checks of the strip partition's host logic, no GPU:

* msf_strip_bounds (the library's own planner, host-only) partitions the node and element
  columns, keeps the global 4-colour parity (even first local column) and gives every owned
  node its full 3x3 stencil inside the local strip;
* the halo protocol run by two processes over torch.distributed (gloo, world_size 2): each
  rank fills only its owned columns, exchanges the edge columns the way msf_dist.cu does
  (first owned column -> left neighbour's right halo, last owned column -> right
  neighbour's left halo), applies the operator assembled from ITS strip's elements only
  (oracle/fem.py), and the owned rows plus the all-reduced dot product equal the
  whole-grid operator's."""
import os
import socket

import numpy as np
import pytest

import workloads as W
from oracle import fem


@pytest.fixture(scope="module")
def pkg():
    from paper_1411_3923_b200 import build
    build.build()
    import paper_1411_3923_b200 as p
    p.load_library()
    return p


@pytest.mark.parametrize("nelx,cx,nranks", [(16, 4, 2), (16, 4, 4), (30, 3, 3), (30, 3, 4),
                                            (36, 4, 3), (32, 8, 3), (60, 20, 3), (54, 9, 2), (1024, 16, 8),
                                            (5120, 20, 8)])
def test_strip_bounds(pkg, nelx, cx, nranks):
    spec = W.small_spec(nelx=nelx, nely=8, cx=cx, cy=4)
    prob = pkg.problem_from_spec(spec)
    owned = np.zeros(nelx + 1, dtype=int)
    elems = np.zeros(nelx, dtype=int)
    # halo width: 8 node columns per side (the streaming sweep's dependency
    # halo) when every strip is at least 8 columns wide, else one column (colour-phase sweep)
    ncx = nelx // cx
    minw = min(((r + 1) * ncx // nranks - r * ncx // nranks) * cx for r in range(nranks))
    h = 8 if minw >= 8 else 1
    for r in range(nranks):
        b = pkg.strip_bounds(prob, r, nranks)
        owned[b["own0"]:b["own1"]] += 1
        elems[b["e0"]:b["e1"]] += 1
        assert b["gox"] % 2 == 0                         # colour parity of the global grid
        lo, hi = b["gox"], b["gox"] + b["ncols"]          # local node columns [lo, hi)
        assert lo <= max(b["own0"] - h, 0) and hi >= min(b["own1"] + h, nelx + 1)
        assert b["own0"] - lo <= h + 1 and hi - b["own1"] <= h   # at most padding + halo
        if r > 0:
            assert b["own0"] - lo >= h
        if r < nranks - 1:
            assert hi - b["own1"] == h
        assert b["e0"] == b["C0"] * cx and b["e1"] == b["C1"] * cx
        assert b["C1"] > b["C0"]
    assert (owned == 1).all() and (elems == 1).all()


def test_strip_bounds_rejects(pkg):
    prob = pkg.problem_from_spec(W.small_spec(nelx=16, nely=8, cx=4, cy=4))
    with pytest.raises(RuntimeError, match="ncx"):
        pkg.strip_bounds(prob, 0, 5)
    with pytest.raises(RuntimeError, match="rank"):
        pkg.strip_bounds(prob, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _halo_worker(rank, world, port, bounds, spec_kw, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec = W.small_spec(**spec_kw)
        nny = spec.nely + 1
        rng = np.random.default_rng(5)
        E = 1e-3 + rng.random(spec.n_el)
        xg = rng.standard_normal((spec.nelx + 1) * nny * 2)
        fx = W.fixed_mask(spec)
        xg[fx.astype(bool)] = 0.0
        b = bounds[rank]
        lo, n = b["gox"], b["ncols"]
        o0, o1 = b["own0"] - lo, b["own1"] - lo
        xl = np.zeros((n, nny, 2))
        xl[o0:o1] = xg.reshape(-1, nny, 2)[b["own0"]:b["own1"]]
        col = lambda i: torch.from_numpy(np.ascontiguousarray(xl[i]))
        reqs, recv = [], {}
        if rank > 0:
            reqs.append(dist.isend(col(o0), rank - 1))
            recv[o0 - 1] = torch.empty(nny, 2, dtype=torch.float64)
            reqs.append(dist.irecv(recv[o0 - 1], rank - 1))
        if rank < world - 1:
            reqs.append(dist.isend(col(o1 - 1), rank + 1))
            recv[o1] = torch.empty(nny, 2, dtype=torch.float64)
            reqs.append(dist.irecv(recv[o1], rank + 1))
        for rq in reqs:
            rq.wait()
        for i, t in recv.items():
            xl[i] = t.numpy()
        # operator of the strip's own elements, Dirichlet rows/cols of the owned nodes
        K0 = fem.element_stiffness(spec.nu)
        El = E[lo * spec.nely:(lo + n - 1) * spec.nely]
        Kl = fem.assemble(n - 1, spec.nely, El, K0)
        fl = fx.reshape(-1, nny, 2)[lo:lo + n].reshape(-1)
        yl = (Kl @ xl.reshape(-1)).reshape(n, nny, 2)
        yl[fl.reshape(n, nny, 2).astype(bool)] = 0.0
        owned_y = yl[o0:o1].copy()
        dot = torch.tensor([float(np.sum(xl[o0:o1] * owned_y))], dtype=torch.float64)
        dist.all_reduce(dot)
        out_q.put((rank, b["own0"], owned_y, float(dot[0]), xl))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("spec_kw", [dict(nelx=16, nely=8, cx=4, cy=4, seed=3),
                                     dict(nelx=18, nely=6, cx=3, cy=3, seed=4)])
def test_gloo_halo_protocol_world2(pkg, spec_kw):
    import torch.multiprocessing as mp
    spec = W.small_spec(**spec_kw)
    prob = pkg.problem_from_spec(spec)
    world = 2
    bounds = [pkg.strip_bounds(prob, r, world) for r in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, bounds, spec_kw, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # whole-grid reference
    nny = spec.nely + 1
    rng = np.random.default_rng(5)
    E = 1e-3 + rng.random(spec.n_el)
    xg = rng.standard_normal((spec.nelx + 1) * nny * 2)
    fx = W.fixed_mask(spec)
    xg[fx.astype(bool)] = 0.0
    A = fem.constrained_operator(fem.assemble(spec.nelx, spec.nely, E,
                                              fem.element_stiffness(spec.nu)), fx)
    yg = (A @ xg).reshape(-1, nny, 2)
    dot_ref = float(xg @ (A @ xg))
    for rank, own0, owned_y, dot, xl in res:
        b = bounds[rank]
        np.testing.assert_allclose(owned_y, yg[own0:own0 + owned_y.shape[0]], rtol=0,
                                   atol=1e-12 * np.abs(yg).max())
        # after the exchange the local strip holds the global field on owned + halo columns
        lo = b["gox"]
        h0 = max(b["own0"] - 1, 0) - lo
        h1 = min(b["own1"] + 1, spec.nelx + 1) - lo
        np.testing.assert_array_equal(xl[h0:h1], xg.reshape(-1, nny, 2)[lo + h0:lo + h1])
        assert abs(dot - dot_ref) <= 1e-12 * abs(dot_ref)


def _cell_couplings(nbc, m, seed):
    """K_c of a chain of nbc blocks from per-cell SPD couplings [[A_k, B_k], [B_k^T, C_k]]
    (cell k couples blocks k, k+1), like the Galerkin assembly: D_k = C_{k-1} + A_k."""
    rng = np.random.default_rng(seed)
    cells = []
    for _ in range(nbc - 1):
        G = rng.standard_normal((2 * m, 3 * m))
        Kk = G @ G.T + 0.5 * np.eye(2 * m)
        cells.append(Kk)
    K = np.zeros((nbc * m, nbc * m))
    for k, Kk in enumerate(cells):
        K[k * m:(k + 2) * m, k * m:(k + 2) * m] += Kk
    return cells, K


def _coarse_worker(rank, world, port, bounds, nbc, m, seed, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cells, _ = _cell_couplings(nbc, m, seed)
        b_glob = np.random.default_rng(seed + 1).standard_normal(nbc * m)
        C0 = bounds[rank]["C0"]
        C1 = bounds[rank]["C1"] if rank < world - 1 else nbc - 1
        # this rank's chain matrix from ITS cells only (end blocks: partial sums)
        L = C1 - C0 + 1
        M = np.zeros((L * m, L * m))
        for k in range(C0, bounds[rank]["C1"]):
            j = k - C0
            M[j * m:(j + 2) * m, j * m:(j + 2) * m] += cells[k]
        # rhs: interior blocks whole, the chain ends split with the neighbour (restriction partials)
        b = b_glob[C0 * m:(C1 + 1) * m].copy()
        if rank > 0:
            b[:m] *= 0.5
        if rank < world - 1:
            b[-m:] *= 0.5
        ends = np.r_[np.arange(m), np.arange((L - 1) * m, L * m)]
        inner = np.arange(m, (L - 1) * m)
        Mee, Mei, Mii = M[np.ix_(ends, ends)], M[np.ix_(ends, inner)], M[np.ix_(inner, inner)]
        if inner.size:
            S = Mee - Mei @ np.linalg.solve(Mii, Mei.T)
            g = b[ends] - Mei @ np.linalg.solve(Mii, b[inner])
        else:
            S, g = Mee, b[ends]
        # interface system over the nranks + 1 chain ends, all-reduced
        nI = world + 1
        Sg = np.zeros((nI * m, nI * m))
        gg = np.zeros(nI * m)
        idx = np.r_[np.arange(rank * m, (rank + 1) * m), np.arange((rank + 1) * m, (rank + 2) * m)]
        Sg[np.ix_(idx, idx)] = S
        gg[idx] = g
        St, gt = torch.from_numpy(Sg), torch.from_numpy(gg)
        dist.all_reduce(St)
        dist.all_reduce(gt)
        xI = np.linalg.solve(St.numpy(), gt.numpy())
        xe = xI[idx]
        x = np.zeros(L * m)
        x[ends] = xe
        if inner.size:
            x[inner] = np.linalg.solve(Mii, b[inner] - Mei.T @ xe)
        out_q.put((rank, C0, C1, x))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nelx,cx", [(2, 16, 2), (3, 18, 2), (2, 12, 4)])
def test_gloo_distributed_coarse_solve(pkg, world, nelx, cx):
    """The interface decomposition of the distributed K_c: each rank builds
    its chain from its own coarse cells (partial end blocks, split end rhs), reduces it to the
    two ends, the interface system is all-reduced over gloo and solved redundantly, the chain
    is back-substituted; the chains of all ranks equal the dense solve of the whole K_c.
    Chain ends come from the library's strip planner."""
    import torch.multiprocessing as mp
    spec = W.small_spec(nelx=nelx, nely=4, cx=cx, cy=2)
    prob = pkg.problem_from_spec(spec)
    bounds = [pkg.strip_bounds(prob, r, world) for r in range(world)]
    nbc, m = nelx // cx + 1, 3
    _, K = _cell_couplings(nbc, m, seed=11)
    b_glob = np.random.default_rng(12).standard_normal(nbc * m)
    x_ref = np.linalg.solve(K, b_glob)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_coarse_worker, args=(r, world, port, bounds, nbc, m, 11, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    covered = np.zeros(nbc, dtype=int)
    for rank, C0, C1, x in res:
        np.testing.assert_allclose(x, x_ref[C0 * m:(C1 + 1) * m], rtol=0, atol=1e-10 * np.abs(x_ref).max())
        covered[C0:C1 + 1] += 1
    assert (covered >= 1).all()
