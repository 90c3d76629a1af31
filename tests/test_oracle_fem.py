"""Pins of oracle/fem.py against closed forms, invariants and paper-printed sizes."""
import json
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import workloads as W
from oracle import fem

HERE = os.path.dirname(__file__)


def sigmund_closed_form(nu):
    """Published closed-form plane-stress Q4 element matrix (Sigmund 2001, "A 99 line
    topology optimization code", Struct Multidisc Optim 21:120-127), node order
    (0,0),(1,0),(1,1),(0,1).  Independent derivation from the oracle's quadrature."""
    k = [1 / 2 - nu / 6, 1 / 8 + nu / 8, -1 / 4 - nu / 12, -1 / 8 + 3 * nu / 8,
         -1 / 4 + nu / 12, -1 / 8 - nu / 8, nu / 6, 1 / 8 - 3 * nu / 8]
    idx = [[0, 1, 2, 3, 4, 5, 6, 7], [1, 0, 7, 6, 5, 4, 3, 2], [2, 7, 0, 5, 6, 3, 4, 1],
           [3, 6, 5, 0, 7, 2, 1, 4], [4, 5, 6, 7, 0, 1, 2, 3], [5, 4, 3, 2, 1, 0, 7, 6],
           [6, 3, 4, 1, 2, 7, 0, 5], [7, 2, 1, 4, 3, 6, 5, 0]]
    return np.array([[k[j] for j in row] for row in idx]) / (1 - nu * nu)


@pytest.mark.parametrize("nu", [0.0, 0.25, 0.3, 0.45])
def test_K0_matches_published_closed_form(nu):
    assert np.abs(fem.element_stiffness(nu) - sigmund_closed_form(nu)).max() < 1e-14


def test_K0_spec_example_entry():
    nu = 0.3
    assert abs(fem.element_stiffness(nu)[0, 0] - (1 / (1 - nu ** 2)) * (0.5 - nu / 6)) < 1e-15


def rigid_modes(x, y):
    """Translations x, y and the infinitesimal rotation at node coordinates."""
    n = x.size
    t1 = np.zeros(2 * n); t1[0::2] = 1
    t2 = np.zeros(2 * n); t2[1::2] = 1
    rot = np.zeros(2 * n); rot[0::2] = -y; rot[1::2] = x
    return np.stack([t1, t2, rot])


def test_K0_rigid_body_null_space_and_psd():
    K0 = fem.element_stiffness(0.3)
    assert np.abs(K0 - K0.T).max() < 1e-16 * 8
    ev = np.linalg.eigvalsh(K0)
    assert (np.abs(ev) < 1e-12 * ev.max()).sum() == 3
    assert ev.min() > -1e-14
    x = np.array([0, 1, 1, 0.0]); y = np.array([0, 0, 1, 1.0])
    for v in rigid_modes(x, y):
        assert np.abs(K0 @ v).max() < 1e-14


def test_patch_test_linear_field():
    """Q4 patch test: a linear displacement field produces zero internal force at every
    interior node of a uniform patch and strain energy = area * eps^T C eps / 2 * 2."""
    nelx, nely, nu = 5, 4, 0.3
    K = fem.assemble(nelx, nely, np.ones(nelx * nely), fem.element_stiffness(nu))
    ix, iy = np.meshgrid(np.arange(nelx + 1), np.arange(nely + 1), indexing="ij")
    x, y = ix.ravel().astype(float), iy.ravel().astype(float)
    a, b, c, d = 0.3, -0.2, 0.15, 0.4
    u = np.zeros(2 * x.size); u[0::2] = a * x + b * y; u[1::2] = c * x + d * y
    Ku = K @ u
    interior = ((ix > 0) & (ix < nelx) & (iy > 0) & (iy < nely)).ravel()
    assert np.abs(Ku.reshape(-1, 2)[interior]).max() < 1e-13
    eps = np.array([a, d, b + c])
    energy = nelx * nely * eps @ fem.plane_stress_C(nu) @ eps
    assert abs(u @ Ku - energy) < 1e-12 * energy


def test_assembled_K_symmetric_spd_and_rigid_null_space():
    s = W.small_spec(nelx=6, nely=4, cx=2, cy=2)
    E = fem.simp_modulus(W.design_tile(s), s.E0, s.Emin, s.penal)
    K = fem.assemble(s.nelx, s.nely, E, fem.element_stiffness(s.nu))
    Kd = K.toarray()
    assert np.abs(Kd - Kd.T).max() < 1e-15 * np.abs(Kd).max()
    ix, iy = np.meshgrid(np.arange(s.nelx + 1), np.arange(s.nely + 1), indexing="ij")
    for v in rigid_modes(ix.ravel().astype(float), iy.ravel().astype(float)):
        assert np.abs(Kd @ v).max() < 1e-12 * np.abs(Kd).max()
    free = W.fixed_mask(s) == 0
    Kff = Kd[np.ix_(free, free)]
    np.linalg.cholesky(Kff)                        # SPD once supports are applied


def test_assembly_equals_brute_force_loop():
    nelx, nely = 3, 2
    E = np.array([1.0, 0.5, 2.0, 1e-3, 0.7, 3.0])
    K0 = fem.element_stiffness(0.3)
    n = 2 * (nelx + 1) * (nely + 1)
    Kb = np.zeros((n, n))
    for ex in range(nelx):
        for ey in range(nely):
            nodes = [ex * (nely + 1) + ey, (ex + 1) * (nely + 1) + ey,
                     (ex + 1) * (nely + 1) + ey + 1, ex * (nely + 1) + ey + 1]
            dofs = [2 * m + c for m in nodes for c in (0, 1)]
            for i in range(8):
                for j in range(8):
                    Kb[dofs[i], dofs[j]] += E[ex * nely + ey] * K0[i, j]
    assert np.abs(fem.assemble(nelx, nely, E, K0).toarray() - Kb).max() < 1e-15


def test_simp_endpoints():
    assert fem.simp_modulus(np.array(0.0), 1.0, 1e-9, 3) == 1e-9
    assert fem.simp_modulus(np.array(1.0), 1.0, 1e-9, 3) == 1.0
    assert fem.simp_modulus(np.array(0.5), 1.0, 0.0, 3) == 0.125


def test_direct_solve_compliance_identities():
    s = W.small_spec(nelx=8, nely=4, cx=4, cy=2)
    fx, f = W.fixed_mask(s), W.load_vector(s)
    E = fem.simp_modulus(W.design_tile(s), s.E0, s.Emin, s.penal)
    K0 = fem.element_stiffness(s.nu)
    K = fem.assemble(s.nelx, s.nely, E, K0)
    u = fem.solve_direct(K, f, fx)
    assert np.all(u[fx == 1] == 0)
    A = fem.constrained_operator(K, fx)
    assert np.linalg.norm(A @ u - f) < 1e-8 * np.linalg.norm(f) * 1e3
    c = fem.compliance(f, u)
    assert c > 0 and abs(c - u @ (K @ u)) < 1e-10 * c
    assert abs(c - fem.element_energy(s.nelx, s.nely, u, K0) @ E) < 1e-10 * c
    # linearity in the modulus: doubling every E halves the displacement
    u2 = fem.solve_direct(fem.assemble(s.nelx, s.nely, 2 * E, K0), f, fx)
    assert np.abs(u2 - 0.5 * u).max() < 1e-9 * np.abs(u).max()


def test_dense_oracle_small_solve():
    s = W.small_spec(nelx=2, nely=2, cx=1, cy=1, design="iid")
    fx, f = W.fixed_mask(s), W.load_vector(s)
    E = np.ones(4)
    K = fem.assemble(2, 2, E, fem.element_stiffness(0.3)).toarray()
    free = fx == 0
    ud = np.zeros_like(f)
    ud[free] = np.linalg.solve(K[np.ix_(free, free)], f[free])
    u = fem.solve_direct(fem.assemble(2, 2, E, fem.element_stiffness(0.3)), f, fx)
    assert np.abs(u - ud).max() < 1e-12 * np.abs(ud).max()


def test_paper_printed_sizes():
    g = json.load(open(os.path.join(HERE, "golden", "paper_sizes.json")))
    for case in g["cases"]:
        nelx, nely = case["nelx"], case["nely"]
        assert nelx == case["coarse_x"] * case["fine_per_coarse"]
        assert nely == case["coarse_y"] * case["fine_per_coarse"]
        assert nelx * nely == case["n_elements"]
        spec = W.small_spec(nelx=nelx, nely=nely, cx=case["fine_per_coarse"],
                            cy=case["fine_per_coarse"])
        if "n_dof" in case:
            assert spec.n_dof == case["n_dof"]
        assert fem.element_dofs(3, 2).max() == 2 * 4 * 3 - 1


def test_baseline_config_dofs():
    # BASELINE configs[0] prints "96x48 elements (9,898 DOF)"; a 96x48 Q4 grid has
    # 2*97*49 = 9,506 DOF (9,898 = 2*101*49 would be 100x48, not divisible by the 8x8
    # coarse cells).  DESIGN.md reading R12: the element grid wins.
    assert W.CONFIGS["c0_cantilever_96x48"].n_dof == 9506
    assert W.CONFIGS["c4_mbb_5120x2560"].n_dof == 26229762       # ~26.2M DOF
