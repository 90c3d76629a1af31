"""ORACLE (test infrastructure only) -- spectral MsFEM coarse space and the two-level
preconditioner.

PAPER.md §2.4 (lines 104-138):
  * coarse mesh T^H obtained by refinement; coarse nodes y_i; agglomerate
    omega_i = union of closed coarse cells containing y_i (line 118);
  * local generalised eigenproblem K_omega psi = lambda M_omega psi (Eq. 9),
    local matrices "take the physical boundary conditions of the full problem into
    account" (line 130), interior agglomerates are "unconstrained and allowing rigid body
    motion" (§2.4.1) -> Neumann assembly over the elements of omega_i;
  * weighting matrix M_omega = diag(K_omega) (§3.2: "use the diagonal of the
    agglomerate stiffness matrix as the weighting matrix");
  * coarse basis phi_{i,j} = psi_j^{omega_i} chi_i with a partition of unity chi_i,
    |grad chi_i| <= 1/H (line 132) -> bilinear coarse hat functions (reading R6);
  * K_c = R_c K R_c^T, f_c = R_c f (Eq. 10); R_c^T = [phi_1 ... phi_Nt].
PAPER.md §2.4.2 (line 146): coarse correction "combined with a single pre- and
post-smoothing using symmetric Gauss-Seidel" -> V-cycle preconditioner.

Readings: R5 a fixed number n_modes of eigenpairs per agglomerate (the
BASELINE configs fix the count instead of a threshold lambda_Omega); R6 chi_i is the
bilinear hat of coarse node i evaluated at fine nodes; R7 the Gauss-Seidel DOF order is
the 4-colour node order (colour = (ix%2) + 2*(iy%2)), x-component before y-component
within a node (the paper does not state an order); R8 "single pre- and post-smoothing
using symmetric Gauss-Seidel" = one symmetric sweep (forward then backward) before and one
after the coarse correction.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from . import fem


# ------------------------------------------------------------------ agglomerates (§2.4)
def coarse_grid(nelx, nely, cx, cy):
    assert nelx % cx == 0 and nely % cy == 0
    return nelx // cx, nely // cy


def agglomerate_box(I, J, nelx, nely, cx, cy):
    """Element box [ex0, ex1) x [ey0, ey1) of omega_{I,J} = union of the (up to 4) coarse
    cells having coarse node (I, J) as a vertex."""
    ex0, ex1 = max(0, (I - 1) * cx), min(nelx, (I + 1) * cx)
    ey0, ey1 = max(0, (J - 1) * cy), min(nely, (J + 1) * cy)
    return ex0, ex1, ey0, ey1


def local_problem(I, J, nelx, nely, cx, cy, E, K0, fixed):
    """K_omega and its diagonal D on the free local DOFs of omega_{I,J} (Eq. 9 with
    the §3.2 diagonal weighting).  Returns (K_loc dense, D, global dof ids of the free
    local DOFs, node coordinates ix, iy of those DOFs)."""
    ex0, ex1, ey0, ey1 = agglomerate_box(I, J, nelx, nely, cx, cy)
    nx, ny = ex1 - ex0, ey1 - ey0
    nloc = 2 * (nx + 1) * (ny + 1)
    Kl = np.zeros((nloc, nloc))
    for ex in range(ex0, ex1):
        for ey in range(ey0, ey1):
            lx, ly = ex - ex0, ey - ey0
            ln = [lx * (ny + 1) + ly, (lx + 1) * (ny + 1) + ly,
                  (lx + 1) * (ny + 1) + ly + 1, lx * (ny + 1) + ly + 1]
            ld = np.array([[2 * n, 2 * n + 1] for n in ln]).ravel()
            Kl[np.ix_(ld, ld)] += E[ex * nely + ey] * K0
    lix, liy = np.meshgrid(np.arange(ex0, ex1 + 1), np.arange(ey0, ey1 + 1), indexing="ij")
    gnode = (lix * (nely + 1) + liy).ravel()
    gdof = np.stack([2 * gnode, 2 * gnode + 1], axis=1).ravel()
    dix = np.repeat(lix.ravel(), 2)
    diy = np.repeat(liy.ravel(), 2)
    keep = fixed[gdof] == 0
    Kf = Kl[np.ix_(keep, keep)]
    return Kf, np.diag(Kf).copy(), gdof[keep], dix[keep], diy[keep]


def local_eigenpairs(Kl, D, n_modes, lam_threshold=np.inf):
    """Smallest eigenpairs of K_omega psi = lambda diag(K_omega) psi (Eq. 9, §3.2),
    psi normalised psi^T D psi = 1, eigenvalues ascending (line 132).  Keeps the first
    n_modes, and of those only eigenvalues < lambda_Omega (line 132: "N_i is determined as
    the number of eigenvalues smaller than a globally selected threshold value"); reading
    R5: n_modes is a cap, lam_threshold = inf gives a fixed count."""
    k = min(n_modes, Kl.shape[0])
    if k == 0:
        return np.zeros(0), np.zeros((Kl.shape[0], 0))
    lam, psi = sla.eigh(Kl, np.diag(D), subset_by_index=[0, k - 1])
    keep = lam < lam_threshold
    return lam[keep], psi[:, keep]


def partition_of_unity(I, J, ix, iy, cx, cy):
    """chi_{I,J} at fine nodes: bilinear coarse hat (reading R6; sum_i chi_i = 1,
    |grad chi_i| <= 1/H)."""
    return (np.maximum(0.0, 1.0 - np.abs(ix - I * cx) / cx)
            * np.maximum(0.0, 1.0 - np.abs(iy - J * cy) / cy))


def build_coarse_basis(nelx, nely, cx, cy, n_modes, E_basis, K0, fixed,
                       lam_threshold=np.inf):
    """R_c (Nt x n_dof, sparse) with rows phi_{i,j} = chi_i psi_j^{omega_i} (PAPER.md
    lines 132-138), rows ordered by coarse node (I*(ncy+1)+J) then mode; also returns the
    kept eigenvalues per agglomerate."""
    ncx, ncy = coarse_grid(nelx, nely, cx, cy)
    n_dof = 2 * (nelx + 1) * (nely + 1)
    rows, cols, vals = [], [], []
    eigvals = {}
    Nt = 0
    for I in range(ncx + 1):
        for J in range(ncy + 1):
            Kl, D, gdof, dix, diy = local_problem(I, J, nelx, nely, cx, cy, E_basis, K0, fixed)
            lam, psi = local_eigenpairs(Kl, D, n_modes, lam_threshold)
            eigvals[(I, J)] = lam
            chi = partition_of_unity(I, J, dix, diy, cx, cy)
            for a in range(psi.shape[1]):
                v = chi * psi[:, a]
                nz = v != 0.0
                rows.append(np.full(nz.sum(), Nt))
                cols.append(gdof[nz])
                vals.append(v[nz])
                Nt += 1
    R = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                      shape=(Nt, n_dof)).tocsr()
    return R, eigvals


def coarse_matrix(R, A):
    """K_c = R_c K R_c^T (Eq. 10), dense."""
    return (R @ A @ R.T).toarray()


# ------------------------------------------------------------------ smoother (§2.4.2)
def gs_groups(nelx, nely, fixed):
    """DOF groups of reading R7 in forward order: colour c = (ix%2) + 2*(iy%2) for
    c = 0..3, within a colour all x-DOFs then all y-DOFs.  DOFs inside one group are
    mutually uncoupled (pinned by tests), so updating a whole group at once equals
    visiting its DOFs one by one."""
    ix, iy = np.meshgrid(np.arange(nelx + 1), np.arange(nely + 1), indexing="ij")
    node = (ix * (nely + 1) + iy).ravel()
    colour = ((ix % 2) + 2 * (iy % 2)).ravel()
    groups = []
    for c in range(4):
        nodes = node[colour == c]
        for comp in (0, 1):
            d = 2 * nodes + comp
            d = d[fixed[d] == 0]
            groups.append(np.sort(d))
    return groups


def gauss_seidel(A, z, r, groups, backward=False):
    """One Gauss-Seidel sweep on A z = r in the order of ``groups`` (reversed when
    backward): z_i += (r_i - (A z)_i) / A_ii."""
    z = z.copy()
    diag = A.diagonal()
    order = groups[::-1] if backward else groups
    for g in order:
        z[g] += (r[g] - A[g] @ z) / diag[g]
    return z


def symmetric_gauss_seidel(A, z, r, groups):
    """Symmetric GS: forward sweep then backward sweep."""
    return gauss_seidel(A, gauss_seidel(A, z, r, groups), r, groups, backward=True)


class TwoLevelPreconditioner:
    """PAPER.md §2.4.2 (line 146): "The residual of the fine-scale system is restricted to
    the coarse basis and the correction is approximated using a MsFEM coarse-scale solve and
    projected back to the fine space ... combined with a single pre- and post-smoothing
    using symmetric Gauss-Seidel".  Reading R8:
        z1 = SGS(0; r);  z2 = z1 + R^T K_c^{-1} R (r - A z1);  z = SGS(z2; r)."""

    def __init__(self, A, R, groups, fixed):
        self.A, self.R, self.groups, self.fixed = A, R, groups, fixed
        self.Kc = coarse_matrix(R, A)
        self.Kc_cho = sla.cho_factor(self.Kc)

    def coarse_correction(self, t):
        return self.R.T @ sla.cho_solve(self.Kc_cho, self.R @ t)

    def __call__(self, r):
        z = symmetric_gauss_seidel(self.A, np.zeros_like(r), r, self.groups)
        z = z + self.coarse_correction(r - self.A @ z)
        z = symmetric_gauss_seidel(self.A, z, r, self.groups)
        z[self.fixed != 0] = 0.0
        return z
