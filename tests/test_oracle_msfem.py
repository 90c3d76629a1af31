"""Pins of oracle/msfem.py and oracle/pcg.py: partition of unity, local spectra,
Gauss-Seidel vs brute force, Galerkin identities, preconditioner symmetry/definiteness,
PCG vs direct solve, contrast-flat iteration counts."""
import numpy as np
import pytest
import scipy.sparse as sp

import workloads as W
from oracle import fem, msfem, pcg, problem


def setup(spec, x=None):
    fx, f = W.fixed_mask(spec), W.load_vector(spec)
    x = W.design_tile(spec) if x is None else x
    K0 = fem.element_stiffness(spec.nu)
    _, _, _, E = problem.element_moduli(spec, x)
    A = fem.constrained_operator(fem.assemble(spec.nelx, spec.nely, E[0], K0), fx)
    return fx, f, K0, E, A


def test_partition_of_unity():
    nelx, nely, cx, cy = 12, 8, 4, 4
    ncx, ncy = msfem.coarse_grid(nelx, nely, cx, cy)
    ix, iy = np.meshgrid(np.arange(nelx + 1), np.arange(nely + 1), indexing="ij")
    ix, iy = ix.ravel(), iy.ravel()
    tot = np.zeros(ix.size)
    for I in range(ncx + 1):
        for J in range(ncy + 1):
            chi = msfem.partition_of_unity(I, J, ix, iy, cx, cy)
            assert chi.min() >= 0 and chi.max() <= 1
            ex0, ex1, ey0, ey1 = msfem.agglomerate_box(I, J, nelx, nely, cx, cy)
            inside = (ix >= ex0) & (ix <= ex1) & (iy >= ey0) & (iy <= ey1)
            assert np.all(chi[~inside] == 0)                 # support in omega_i
            # |grad chi| <= 1/H along grid lines
            C = chi.reshape(nelx + 1, nely + 1)
            assert np.abs(np.diff(C, axis=0)).max() <= 1 / cx + 1e-15
            tot += chi
    assert np.abs(tot - 1).max() < 1e-15


def test_agglomerate_boxes():
    nelx, nely, cx, cy = 12, 8, 4, 4
    assert msfem.agglomerate_box(0, 0, nelx, nely, cx, cy) == (0, 4, 0, 4)     # corner: 1 cell
    assert msfem.agglomerate_box(1, 0, nelx, nely, cx, cy) == (0, 8, 0, 4)     # edge: 2 cells
    assert msfem.agglomerate_box(1, 1, nelx, nely, cx, cy) == (0, 8, 0, 8)     # interior: 4
    assert msfem.agglomerate_box(3, 2, nelx, nely, cx, cy) == (8, 12, 4, 8)


def test_interior_agglomerate_rigid_modes_and_clamped_none():
    spec = W.small_spec(nelx=16, nely=8, cx=4, cy=4)
    fx = W.fixed_mask(spec)
    K0 = fem.element_stiffness(spec.nu)
    E = np.ones(spec.n_el)
    Kl, D, gdof, dix, diy = msfem.local_problem(2, 1, spec.nelx, spec.nely, 4, 4, E, K0, fx)
    lam, psi = msfem.local_eigenpairs(Kl, D, 6)
    assert (np.abs(lam) < 1e-12).sum() == 3 and lam[3] > 1e-6
    # the three rigid-body modes lie in the span of the zero-eigenvalue eigenvectors
    x, y = dix[0::2].astype(float), diy[0::2].astype(float)
    Z = psi[:, :3]
    for v in (np.tile([1.0, 0.0], x.size), np.tile([0.0, 1.0], x.size),
              np.ravel(np.stack([-y, x], axis=1))):
        res = v - Z @ np.linalg.lstsq(Z, v, rcond=None)[0]
        assert np.linalg.norm(res) < 1e-10 * np.linalg.norm(v)
    Kc, Dc, *_ = msfem.local_problem(0, 1, spec.nelx, spec.nely, 4, 4, E, K0, fx)
    lamc, _ = msfem.local_eigenpairs(Kc, Dc, 3)
    assert lamc[0] > 1e-4                                                   # clamped: none


def test_local_eigenpairs_residual_orthonormality_and_minimality():
    spec = W.small_spec(nelx=16, nely=8, cx=4, cy=4)
    fx, f, K0, E, A = setup(spec)
    Kl, D, *_ = msfem.local_problem(2, 1, spec.nelx, spec.nely, 4, 4, E[0], K0, fx)
    lam, psi = msfem.local_eigenpairs(Kl, D, 5)
    assert np.all(np.diff(lam) >= 0)
    assert np.abs(psi.T @ (D[:, None] * psi) - np.eye(5)).max() < 1e-10
    res = Kl @ psi - (D[:, None] * psi) * lam[None, :]
    assert np.abs(res).max() < 1e-9 * np.abs(Kl).max()
    # Courant-Fischer: sum of the 5 smallest <= trace of the D-weighted Rayleigh-Ritz
    # projection onto any 5-dim subspace
    rng = np.random.default_rng(0)
    for _ in range(20):
        V = rng.standard_normal((Kl.shape[0], 5))
        G, H = V.T @ Kl @ V, V.T @ (D[:, None] * V)
        assert lam.sum() <= np.trace(np.linalg.solve(H, G)) + 1e-12


def test_threshold_selection():
    spec = W.small_spec(nelx=16, nely=8, cx=4, cy=4)
    fx, f, K0, E, A = setup(spec)
    Kl, D, *_ = msfem.local_problem(2, 1, spec.nelx, spec.nely, 4, 4, E[0], K0, fx)
    lam_all, _ = msfem.local_eigenpairs(Kl, D, 8)
    thr = 0.5 * (lam_all[4] + lam_all[5])
    lam, psi = msfem.local_eigenpairs(Kl, D, 8, thr)
    assert lam.size == 5 and psi.shape[1] == 5


def test_gs_groups_uncoupled_and_cover_free_dofs():
    spec = W.small_spec(nelx=6, nely=5, cx=3, cy=5)
    fx, f, K0, E, A = setup(spec)
    groups = msfem.gs_groups(spec.nelx, spec.nely, fx)
    allg = np.concatenate(groups)
    assert np.array_equal(np.sort(allg), np.flatnonzero(fx == 0))
    for g in groups:
        B = A[g][:, g].toarray()
        assert np.count_nonzero(B - np.diag(np.diag(B))) == 0


def brute_force_gs(A, z, r, order):
    A = A.toarray()
    z = z.copy()
    for i in order:
        z[i] += (r[i] - A[i] @ z) / A[i, i]
    return z


def test_gauss_seidel_equals_sequential_dof_loop():
    spec = W.small_spec(nelx=6, nely=4, cx=3, cy=2)
    fx, f, K0, E, A = setup(spec)
    groups = msfem.gs_groups(spec.nelx, spec.nely, fx)
    order = np.concatenate(groups)
    rng = np.random.default_rng(1)
    r = rng.standard_normal(spec.n_dof); r[fx == 1] = 0
    z0 = rng.standard_normal(spec.n_dof); z0[fx == 1] = 0
    zf = msfem.gauss_seidel(A, z0, r, groups)
    assert np.abs(zf - brute_force_gs(A, z0, r, order)).max() < 1e-12 * np.abs(zf).max()
    zb = msfem.gauss_seidel(A, z0, r, groups, backward=True)
    assert np.abs(zb - brute_force_gs(A, z0, r, order[::-1])).max() < 1e-12 * np.abs(zb).max()


def test_sgs_and_two_level_preconditioner_spd():
    spec = W.small_spec(nelx=16, nely=8, cx=4, cy=4)
    fx, f, K0, E, A = setup(spec)
    R, _ = msfem.build_coarse_basis(spec.nelx, spec.nely, 4, 4, 4, E[0], K0, fx)
    groups = msfem.gs_groups(spec.nelx, spec.nely, fx)
    M = msfem.TwoLevelPreconditioner(A, R, groups, fx)
    rng = np.random.default_rng(2)
    V = rng.standard_normal((6, spec.n_dof)); V[:, fx == 1] = 0
    Z = np.array([M(v) for v in V])
    S = np.array([msfem.symmetric_gauss_seidel(A, np.zeros(spec.n_dof), v, groups) for v in V])
    for i in range(6):
        assert Z[i] @ V[i] > 0
        for j in range(i):
            assert abs(Z[i] @ V[j] - Z[j] @ V[i]) < 1e-10 * abs(Z[i] @ V[j])
            assert abs(S[i] @ V[j] - S[j] @ V[i]) < 1e-10 * abs(S[i] @ V[j])
    assert np.array_equal(M(np.zeros(spec.n_dof)), np.zeros(spec.n_dof))


def test_galerkin_coarse_matrix_and_projector():
    spec = W.small_spec(nelx=12, nely=8, cx=4, cy=4)
    fx, f, K0, E, A = setup(spec)
    R, _ = msfem.build_coarse_basis(spec.nelx, spec.nely, 4, 4, 3, E[0], K0, fx)
    Kc = msfem.coarse_matrix(R, A)
    Rd = R.toarray()
    # entries equal phi_a^T K phi_b from dense vectors (different route than R A R^T)
    Kd = A.toarray()
    for a, b in [(0, 0), (3, 7), (10, 2), (Rd.shape[0] - 1, 5)]:
        assert abs(Kc[a, b] - Rd[a] @ Kd @ Rd[b]) < 1e-12 * np.abs(Kc).max()
    assert np.abs(Kc - Kc.T).max() < 1e-13 * np.abs(Kc).max()
    np.linalg.cholesky(Kc)
    # coarse correction C = R^T Kc^-1 R is the A-orthogonal projector onto span(R^T)
    M = msfem.TwoLevelPreconditioner(A, R, msfem.gs_groups(spec.nelx, spec.nely, fx), fx)
    c = np.random.default_rng(3).standard_normal(Rd.shape[0])
    v = R.T @ c
    assert np.linalg.norm(M.coarse_correction(A @ v) - v) < 1e-9 * np.linalg.norm(v)
    # Galerkin orthogonality: R (A e) = 0 for the error of the coarse solution
    u = fem.solve_direct(fem.assemble(spec.nelx, spec.nely, E[0], K0), f, fx)
    ua = M.coarse_correction(f)
    assert np.abs(R @ (A @ (u - ua))).max() < 1e-8 * np.abs(R @ f).max()
    # energy error < 1 (§3.1: relative energy norm error of a single MsFEM solve)
    e = u - ua
    assert (e @ A @ e) / (u @ A @ u) < 1.0


@pytest.mark.parametrize("bc", ["cantilever", "mbb"])
def test_pcg_matches_direct_solve(bc):
    spec = W.small_spec(nelx=16, nely=8, cx=4, cy=4, bc=bc, Emin=1e-6)
    fx, f = W.fixed_mask(spec), W.load_vector(spec)
    out = problem.solve(spec, W.design_tile(spec), fx, f, tol=1e-12)
    ud = fem.solve_direct(fem.assemble(spec.nelx, spec.nely, out["E_el"][0], out["K0"]), f, fx)
    assert np.linalg.norm(out["us"][0] - ud) < 1e-8 * np.linalg.norm(ud)
    assert out["iters"][0] < 100


def test_pcg_textbook_cases():
    Aid = lambda v: v
    f = np.arange(1.0, 6.0)
    x, it, _ = pcg.pcg(Aid, f, lambda r: r, tol=1e-12)
    assert it == 1 and np.allclose(x, f)
    x, it, _ = pcg.pcg(Aid, np.zeros(5), lambda r: r)
    assert it == 0 and np.all(x == 0)
    # CG terminates in at most n steps on an SPD n x n system
    rng = np.random.default_rng(4)
    B = rng.standard_normal((8, 8)); S = B @ B.T + 8 * np.eye(8)
    x, it, _ = pcg.pcg(lambda v: S @ v, f[:5].repeat(2)[:8], lambda r: r, tol=1e-12)
    assert it <= 8 and np.linalg.norm(S @ x - f[:5].repeat(2)[:8]) < 1e-10 * 10


def test_contrast_flat_iterations():
    """North star invariant: PCG iteration counts stay nearly flat as the stiffness
    contrast grows (§3.1 line 197 'clear contrast-independence')."""
    base = W.small_spec(nelx=48, nely=24, cx=8, cy=8, n_modes=4, design="iid", seed=11)
    x = W.design_tile(base)
    fx, f = W.fixed_mask(base), W.load_vector(base)
    its = {}
    for Emin in (1e0, 1e-3, 1e-6, 1e-9):
        spec = base.replace(Emin=Emin, E0=2.0 if Emin == 1.0 else 1.0)
        its[Emin] = problem.solve(spec, x, fx, f)["iters"][0]
    hi = [its[e] for e in (1e-3, 1e-6, 1e-9)]
    assert max(hi) - min(hi) <= 0.1 * max(hi) + 1
    assert its[1e0] <= min(hi)


# ---------------------------------------------------------------- round-2 pins
def test_local_problem_moduli_mapping_brute_force():
    """Pin of local_problem's element-moduli mapping (Eq. 9, l.128-130: K_omega is
    the stiffness of the elements of omega_i).  Brute force: assemble the WHOLE grid with
    the moduli zeroed outside the agglomerate box; its rows/columns of the box DOFs must be
    K_omega.  The grid is non-square and E heterogeneous, so a transposed E index, a
    shifted box or a wrong local node order all fail."""
    nelx, nely, cx, cy = 12, 6, 4, 3
    K0 = fem.element_stiffness(0.3)
    rng = np.random.default_rng(21)
    E = rng.uniform(0.1, 2.0, nelx * nely)
    fixed = np.zeros(2 * (nelx + 1) * (nely + 1), dtype=np.int8)
    ex, ey = np.meshgrid(np.arange(nelx), np.arange(nely), indexing="ij")
    ex, ey = ex.ravel(), ey.ravel()                     # element id = ex*nely + ey
    for (I, J) in [(0, 0), (1, 1), (3, 2), (2, 0)]:
        ex0, ex1, ey0, ey1 = msfem.agglomerate_box(I, J, nelx, nely, cx, cy)
        inside = (ex >= ex0) & (ex < ex1) & (ey >= ey0) & (ey < ey1)
        Kg = fem.assemble(nelx, nely, np.where(inside, E, 0.0), K0).toarray()
        Kl, D, gdof, dix, diy = msfem.local_problem(I, J, nelx, nely, cx, cy, E, K0, fixed)
        assert np.abs(Kl - Kg[np.ix_(gdof, gdof)]).max() < 1e-14 * np.abs(Kg).max()
        # every DOF the box's elements touch is a local DOF
        touched = np.flatnonzero(np.abs(Kg).sum(axis=1) > 0)
        assert set(touched) <= set(gdof)
    # one coarse cell covering the grid: K_omega is the global free-DOF stiffness
    fx = np.zeros(2 * (nelx + 1) * (nely + 1), dtype=np.int8)
    fx[:2 * (nely + 1)] = 1                                # left edge clamped
    Kl, D, gdof, *_ = msfem.local_problem(0, 0, nelx, nely, nelx, nely, E, K0, fx)
    Kg = fem.assemble(nelx, nely, E, K0).toarray()
    free = np.flatnonzero(fx == 0)
    assert np.array_equal(gdof, free)
    assert np.abs(Kl - Kg[np.ix_(free, free)]).max() < 1e-14 * np.abs(Kg).max()


def test_local_eigenpairs_diagonal_weighting():
    """Pin of the §3.2 weighting M_omega = diag(K_omega).
    (a) A one-element agglomerate with nothing fixed: diag(E K0) = E k11 I (the Q4 element
        matrix has one diagonal value), so lambda = eig(K0) / K0[0,0] for every E.
    (b) The pencil (K_omega, diag K_omega) is invariant under E -> alpha E on a
        heterogeneous agglomerate (D = I or D = mass would scale lambda by alpha)."""
    K0 = fem.element_stiffness(0.3)
    assert np.ptp(np.diag(K0)) < 1e-15          # one diagonal value (to rounding)
    ref = np.linalg.eigvalsh(K0) / K0[0, 0]
    nelx, nely = 4, 3
    fixed = np.zeros(2 * (nelx + 1) * (nely + 1), dtype=np.int8)
    for Ev in (1.0, 7.5, 1e-6):
        E = np.full(nelx * nely, Ev)
        Kl, D, *_ = msfem.local_problem(0, 0, nelx, nely, 1, 1, E, K0, fixed)
        assert Kl.shape == (8, 8)
        lam, _ = msfem.local_eigenpairs(Kl, D, 8)
        assert np.abs(lam - ref).max() < 1e-12
    spec = W.small_spec(nelx=16, nely=8, cx=4, cy=4)
    fx = W.fixed_mask(spec)
    E = np.random.default_rng(22).uniform(1e-3, 1.0, spec.n_el)
    lam1 = msfem.local_eigenpairs(*msfem.local_problem(2, 1, 16, 8, 4, 4, E, K0, fx)[:2], 6)[0]
    lam2 = msfem.local_eigenpairs(*msfem.local_problem(2, 1, 16, 8, 4, 4, 300.0 * E, K0, fx)[:2], 6)[0]
    assert np.abs(lam1 - lam2).max() < 1e-10 * max(1.0, np.abs(lam1).max())
    # the weighting is the diagonal itself: Rayleigh quotient of the unit vector e_i is 1
    Kl, D, *_ = msfem.local_problem(2, 1, 16, 8, 4, 4, E, K0, fx)
    assert np.array_equal(D, np.diag(Kl))


def test_coarse_basis_partition_of_unity_weighting():
    """Pin of phi_{i,j} = chi_i psi_j inside build_coarse_basis.
    (a) Rows of R vanish on the nodes of the agglomerate boundary that lie inside the
        domain (chi_i = 0 there; a bare psi does not vanish on a Neumann boundary).
    (b) With no Dirichlet DOFs and uniform E every agglomerate's first 3 modes span the
        rigid-body modes, and sum_i chi_i = 1 makes the three GLOBAL rigid-body modes lie in
        span(R^T) exactly; the unweighted box-restricted modes do not span them.
    (c) On the agglomerate's own coarse node chi = 1 (row = psi there)."""
    nelx, nely, cx, cy = 12, 8, 4, 4
    ncx, ncy = msfem.coarse_grid(nelx, nely, cx, cy)
    K0 = fem.element_stiffness(0.3)
    n_dof = 2 * (nelx + 1) * (nely + 1)
    fixed = np.zeros(n_dof, dtype=np.int8)
    E = np.ones(nelx * nely)
    R, _ = msfem.build_coarse_basis(nelx, nely, cx, cy, 3, E, K0, fixed)
    Rd = R.toarray()
    node_ix = np.repeat(np.arange(nelx + 1), nely + 1)
    node_iy = np.tile(np.arange(nely + 1), nelx + 1)
    dix, diy = np.repeat(node_ix, 2), np.repeat(node_iy, 2)
    row = 0
    for I in range(ncx + 1):
        for J in range(ncy + 1):
            ex0, ex1, ey0, ey1 = msfem.agglomerate_box(I, J, nelx, nely, cx, cy)
            on_bdry = (((dix == ex0) & (ex0 > 0)) | ((dix == ex1) & (ex1 < nelx))
                       | ((diy == ey0) & (ey0 > 0)) | ((diy == ey1) & (ey1 < nely)))
            on_bdry &= (dix >= ex0) & (dix <= ex1) & (diy >= ey0) & (diy <= ey1)
            for _ in range(3):
                assert np.abs(Rd[row, on_bdry]).max() == 0.0
                outside = (dix < ex0) | (dix > ex1) | (diy < ey0) | (diy > ey1)
                assert np.abs(Rd[row, outside]).max() == 0.0
                row += 1
            # (c): at the coarse node, chi = 1 so the row carries psi, which (for the
            # rigid modes of a unit-E agglomerate) does not vanish identically there
            at = (dix == I * cx) & (diy == J * cy)
            assert np.abs(Rd[row - 3:row][:, at]).max() > 0.0
    assert row == Rd.shape[0]
    x, y = node_ix.astype(float), node_iy.astype(float)
    for v in (np.tile([1.0, 0.0], x.size), np.tile([0.0, 1.0], x.size),
              np.ravel(np.stack([-y, x], axis=1))):
        c = np.linalg.lstsq(Rd.T, v, rcond=None)[0]
        assert np.linalg.norm(Rd.T @ c - v) < 1e-10 * np.linalg.norm(v)
