"""ORACLE (test infrastructure only) -- Q4 plane-stress elasticity with modified SIMP.

PAPER.md §2.1 (lines 48-75, Eq. 1-4): linear elasticity, -div sigma = f, sigma = C:eps,
C(x) = E(x) C0 with C0 the isotropic stiffness for unit Young's modulus, discretised
with vector-valued shape functions on a uniform mesh -> K u = f (Eq. 4).
PAPER.md §2.2 (lines 82-86, Eq. 5): K_e(rho_e) = (Emin + (Emax-Emin) rho_e^p) K0.

Readings: R1 plane stress, unit thickness, square unit elements, bilinear Q4
with 2x2 Gauss quadrature; R2 Dirichlet DOFs are eliminated (operator P K P on the free
DOFs, vectors carry zeros on fixed DOFs).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def plane_stress_C(nu: float) -> np.ndarray:
    """C0 for unit Young's modulus, plane stress ("C(x) = E(x) C0 where C0
    is the stiffness tensor for a predefined Poisson's ratio ... and unit Young's modulus";
    reading R1: plane stress)."""
    return (1.0 / (1.0 - nu * nu)) * np.array(
        [[1.0, nu, 0.0], [nu, 1.0, 0.0], [0.0, 0.0, 0.5 * (1.0 - nu)]])


def _dshape(xi: float, eta: float):
    # bilinear shape functions on [-1,1]^2, local nodes (-1,-1),(1,-1),(1,1),(-1,1)
    dxi = 0.25 * np.array([-(1 - eta), (1 - eta), (1 + eta), -(1 + eta)])
    deta = 0.25 * np.array([-(1 - xi), -(1 + xi), (1 + xi), (1 - xi)])
    return dxi, deta


def strain_matrix(xi: float, eta: float, h: float = 1.0) -> np.ndarray:
    """B (3x8) at (xi, eta) for a square element of side h; eps = B u_e."""
    dxi, deta = _dshape(xi, eta)
    dNdx, dNdy = dxi * (2.0 / h), deta * (2.0 / h)
    B = np.zeros((3, 8))
    B[0, 0::2] = dNdx
    B[1, 1::2] = dNdy
    B[2, 0::2] = dNdy
    B[2, 1::2] = dNdx
    return B


def element_stiffness(nu: float, h: float = 1.0) -> np.ndarray:
    """K0 (8x8): a(u,v) = int_e (C0:eps(u)):eps(v) dx (Eq. 3a, line 66) for one
    unit-modulus element, 2x2 Gauss quadrature (exact for the bilinear element).
    Local node order n0=(0,0), n1=(1,0), n2=(1,1), n3=(0,1); DOFs [n0x n0y n1x n1y ...]."""
    C = plane_stress_C(nu)
    g = 1.0 / np.sqrt(3.0)
    detJ = (h / 2.0) ** 2
    K = np.zeros((8, 8))
    for xi in (-g, g):
        for eta in (-g, g):
            B = strain_matrix(xi, eta, h)
            K += B.T @ C @ B * detJ
    return K


def simp_modulus(xbar: np.ndarray, E0: float, Emin: float, p: float) -> np.ndarray:
    """PAPER.md Eq. 5 (line 84): E_e = Emin + (Emax - Emin) rho_e^p."""
    return Emin + np.power(xbar, p) * (E0 - Emin)


def element_dofs(nelx: int, nely: int) -> np.ndarray:
    """(n_el, 8) global DOF ids of each element (element id = ex*nely + ey)."""
    ex, ey = np.meshgrid(np.arange(nelx), np.arange(nely), indexing="ij")
    ex, ey = ex.ravel(), ey.ravel()
    n0 = ex * (nely + 1) + ey
    n1 = (ex + 1) * (nely + 1) + ey
    n2 = (ex + 1) * (nely + 1) + ey + 1
    n3 = ex * (nely + 1) + ey + 1
    nodes = np.stack([n0, n1, n2, n3], axis=1)
    dofs = np.empty((nodes.shape[0], 8), dtype=np.int64)
    dofs[:, 0::2] = 2 * nodes
    dofs[:, 1::2] = 2 * nodes + 1
    return dofs


def assemble(nelx: int, nely: int, E: np.ndarray, K0: np.ndarray) -> sp.csr_matrix:
    """Global stiffness K = sum_e E_e * scatter(K0) (Eq. 4-5), no BCs applied."""
    edofs = element_dofs(nelx, nely)
    rows = np.repeat(edofs, 8, axis=1).ravel()
    cols = np.tile(edofs, (1, 8)).ravel()
    vals = (E[:, None] * K0.ravel()[None, :]).ravel()
    n = 2 * (nelx + 1) * (nely + 1)
    return sp.coo_matrix((vals, (rows, cols)), shape=(n, n)).tocsr()


def constrained_operator(K: sp.csr_matrix, fixed: np.ndarray) -> sp.csr_matrix:
    """A = P K P with P = diag(free): the operator of K u = f on the free DOFs, acting on
    full-length vectors (reading R2)."""
    P = sp.diags((fixed == 0).astype(np.float64))
    return (P @ K @ P).tocsr()


def solve_direct(K: sp.csr_matrix, f: np.ndarray, fixed: np.ndarray) -> np.ndarray:
    """Sparse direct solve on the free DOFs (§4.1: reference results by a
    direct solver)."""
    free = np.flatnonzero(fixed == 0)
    u = np.zeros_like(f)
    Kff = K[free][:, free].tocsc()
    u[free] = spla.spsolve(Kff, f[free])
    return u


def compliance(f: np.ndarray, u: np.ndarray) -> float:
    """PAPER.md Eq. 6 (line 90): c = f^T u."""
    return float(f @ u)


def element_energy(nelx: int, nely: int, u: np.ndarray, K0: np.ndarray) -> np.ndarray:
    """u_e^T K0 u_e per element (the factor in PAPER.md Eq. 14)."""
    ue = u[element_dofs(nelx, nely)]
    return np.einsum("ei,ij,ej->e", ue, K0, ue)
