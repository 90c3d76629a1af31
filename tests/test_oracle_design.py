"""Pins of oracle/design.py: adjoint sensitivities vs finite differences of direct solves,
robust objective hand values, end-to-end tile gradients, OC update feasibility."""
import numpy as np
import pytest

import workloads as W
from oracle import design, fem, filters, problem


def direct_compliances(spec, x_tile, fx, f):
    K0 = fem.element_stiffness(spec.nu)
    _, _, _, E = problem.element_moduli(spec, x_tile)
    us = [fem.solve_direct(fem.assemble(spec.nelx, spec.nely, e, K0), f, fx) for e in E]
    return np.array([fem.compliance(f, u) for u in us]), us, K0


def test_element_sensitivity_fd():
    spec = W.small_spec(nelx=8, nely=4, cx=4, cy=2, Emin=1e-3)
    fx, f = W.fixed_mask(spec), W.load_vector(spec)
    K0 = fem.element_stiffness(spec.nu)
    xb = np.random.default_rng(0).uniform(0.2, 0.9, spec.n_el)

    def comp(x):
        E = fem.simp_modulus(x, spec.E0, spec.Emin, spec.penal)
        u = fem.solve_direct(fem.assemble(spec.nelx, spec.nely, E, K0), f, fx)
        return fem.compliance(f, u), u

    c0, u = comp(xb)
    dc = design.compliance_sensitivity(xb, u, K0, spec.E0, spec.Emin, spec.penal, spec.nelx, spec.nely)
    assert np.all(dc <= 0)
    for e in np.random.default_rng(1).choice(spec.n_el, 10, replace=False):
        h = 1e-4          # central difference: truncation O(h^2) ~ 1e-8, cancellation ~ 1e-9
        xp, xm = xb.copy(), xb.copy()
        xp[e] += h; xm[e] -= h
        fd = (comp(xp)[0] - comp(xm)[0]) / (2 * h)
        assert abs(fd - dc[e]) < 1e-5 * abs(dc[e])
    # rho_e = 0 with p > 1 -> exactly zero sensitivity (rho^{p-1} factor)
    xz = xb.copy(); xz[3] = 0.0
    cz, uz = comp(xz)
    assert design.compliance_sensitivity(xz, uz, K0, spec.E0, spec.Emin, spec.penal,
                                         spec.nelx, spec.nely)[3] == 0.0


def test_robust_objective_hand_values():
    F, mean, var, w = design.robust_objective([2.0, 2.0, 2.0], 1.0)
    assert F == 2.0 and var == 0.0 and np.allclose(w, 1 / 3)
    F, mean, var, w = design.robust_objective([1.0, 2.0, 3.0], 1.0)
    assert abs(mean - 2.0) < 1e-15 and abs(var - 2 / 3) < 1e-15
    assert abs(F - (2.0 + np.sqrt(2 / 3))) < 1e-14
    F0, *_ = design.robust_objective([1.0, 2.0, 3.0], 0.0)
    assert F0 == 2.0
    # dF/dc by finite differences
    c = np.array([1.3, 2.1, 2.9])
    _, _, _, w = design.robust_objective(c, 1.0)
    for k in range(3):
        cp, cm = c.copy(), c.copy()
        cp[k] += 1e-7; cm[k] -= 1e-7
        fd = (design.robust_objective(cp, 1.0)[0] - design.robust_objective(cm, 1.0)[0]) / 2e-7
        assert abs(fd - w[k]) < 1e-7


def test_end_to_end_tile_gradients_fd():
    """F = E[c] + kappa sqrt(Var c) and g through filter -> 3 projections -> tiling ->
    SIMP -> direct solves, differentiated w.r.t. the tile design variables."""
    spec = W.small_spec(nelx=8, nely=8, cx=4, cy=4, tile=(4, 4), rmin=1.5, beta=4.0,
                        etas=(0.7, 0.5, 0.3), dilated=2, Emin=1e-3, volfrac=0.5)
    fx, f = W.fixed_mask(spec), W.load_vector(spec)
    x = np.random.default_rng(2).uniform(0.3, 0.7, 16)
    c, us, K0 = direct_compliances(spec, x, fx, f)
    F, c2, g, dF, dg = design.design_gradients(spec, x, us, f, K0)
    assert np.allclose(c, c2)

    def Fg(xx):
        cc, uu, _ = direct_compliances(spec, xx, fx, f)
        _, xbars = filters.physical_tiles(xx, 4, 4, spec.rmin, spec.beta, spec.etas)
        return (design.robust_objective(cc, spec.kappa)[0],
                design.volume_constraint(xbars, 8, 8, 4, 4, spec.volfrac))

    for i in range(16):
        xp, xm = x.copy(), x.copy()
        xp[i] += 1e-5; xm[i] -= 1e-5
        (Fp, gp), (Fm, gm) = Fg(xp), Fg(xm)
        assert abs((Fp - Fm) / 2e-5 - dF[i]) < 1e-4 * np.abs(dF).max()
        assert abs((gp - gm) / 2e-5 - dg[i]) < 1e-6 * np.abs(dg).max()


def test_volume_constraint_values():
    spec = W.small_spec(nelx=8, nely=8, tile=(4, 4), etas=(0.5,), volfrac=0.5)
    assert design.volume_constraint([np.full(16, 0.5)], 8, 8, 4, 4, 0.5) == 0.0
    assert design.volume_constraint([np.ones(16)], 8, 8, 4, 4, 0.5) == 1.0


def test_oc_update_feasible_and_bounded():
    spec = W.small_spec(nelx=8, nely=8, cx=4, cy=4, tile=(4, 4), rmin=1.5, beta=4.0,
                        etas=(0.7, 0.5, 0.3), dilated=2, Emin=1e-3, volfrac=0.5)
    fx, f = W.fixed_mask(spec), W.load_vector(spec)
    x = np.full(16, 0.5) + np.random.default_rng(3).uniform(-0.1, 0.1, 16)
    c, us, K0 = direct_compliances(spec, x, fx, f)
    F, _, g, dF, dg = design.design_gradients(spec, x, us, f, K0)
    xn = design.oc_update(spec, x, dF, dg)
    assert np.all(xn >= 0) and np.all(xn <= 1) and np.all(np.abs(xn - x) <= 0.2 + 1e-15)
    _, xbars = filters.physical_tiles(xn, 4, 4, spec.rmin, spec.beta, spec.etas)
    assert abs(design.volume_constraint(xbars, 8, 8, 4, 4, spec.volfrac)) < 5e-3
    # the update moves material towards larger -dF/dg ratios
    ratio = -dF / dg
    assert np.corrcoef(ratio, xn - x)[0, 1] > 0
