"""ORACLE (test infrastructure only) -- robust objective, adjoint sensitivities and the
optimality-criteria design update.

PAPER.md §4.2 (lines 245-255): self-adjoint compliance, Eq. 14
  d f / d rho_e = - u_e^T (dK_e/d rho_e) u_e,   Eq. 15  dK_e/d rho_e = p (Emax-Emin) rho_e^{p-1} K0.
PAPER.md §4.3 (line 267): sensitivities corrected by the chain rule through projection and
filter.  PAPER.md §4.1 (line 236): tile-variable sensitivity = sum over controlled elements.
PAPER.md §4.4 Eq. 17 (lines 283-289): f = E[f^T u] + kappa sqrt(Var[f^T u]),
g = E[xbar^T v] / (v_f e^T v) - 1, equal weights, kappa = 1 (line 291).

Readings: R10 population variance with equal weights 1/m; dF/dc_k =
1/m + kappa (c_k - mean) / (m sqrt(Var)) (variance term dropped when Var == 0).
R11 the BASELINE north star replaces MMA (paper §4.1) by the optimality-criteria
update: x_new = clamp(x sqrt(max(0,-dF)/(lambda max(dg,1e-30))), max(0, x-move),
min(1, x+move)), move = 0.2, lambda found by bisection on [0, 1e9] until
(l2-l1)/(l1+l2) < 1e-3 with g evaluated exactly through filter + projections.
"""
from __future__ import annotations

import numpy as np

from . import fem, filters


def compliance_sensitivity(xbar_el, u, K0, E0, Emin, p, nelx, nely):
    """dc/dxbar_e = -p xbar_e^{p-1} (E0-Emin) u_e^T K0 u_e   (Eq. 14-15)."""
    return -p * np.power(xbar_el, p - 1.0) * (E0 - Emin) * fem.element_energy(nelx, nely, u, K0)


def robust_objective(c, kappa):
    """PAPER.md Eq. 17: returns (F, mean, var, dF/dc_k)."""
    c = np.asarray(c, dtype=np.float64)
    m = c.size
    mean = c.mean()
    var = ((c - mean) ** 2).mean()
    w = np.full(m, 1.0 / m)
    if var > 0.0:
        w = w + kappa * (c - mean) / (m * np.sqrt(var))
    return mean + kappa * np.sqrt(var), mean, var, w


def volume_constraint(xbar_tiles, nelx, nely, tile_x, tile_y, volfrac):
    """g = E[xbar^T v]/(v_f e^T v) - 1 with unit element volumes (Eq. 17)."""
    m = len(xbar_tiles)
    tot = 0.0
    for xb in xbar_tiles:
        tot += filters.tile_to_grid(xb, nelx, nely, tile_x, tile_y).sum()
    return tot / (m * nelx * nely * volfrac) - 1.0


def design_gradients(spec, x_tile, us, f, K0):
    """Robust objective F, constraint g and their gradients w.r.t. the tile design
    variables: chain rule through projection (Eq. 16) and density
    filter, summed over the tiling map (line 236)."""
    nelx, nely, tx, ty = spec.nelx, spec.nely, spec.tile_x, spec.tile_y
    xt, xbars = filters.physical_tiles(x_tile, tx, ty, spec.rmin, spec.beta, spec.etas)
    c = np.array([fem.compliance(f, u) for u in us])
    F, mean, var, w = robust_objective(c, spec.kappa)
    m = len(spec.etas)
    dF = np.zeros(tx * ty)
    dg = np.zeros(tx * ty)
    for k, eta in enumerate(spec.etas):
        xb_el = filters.tile_to_grid(xbars[k], nelx, nely, tx, ty)
        dc_el = compliance_sensitivity(xb_el, us[k], K0, spec.E0, spec.Emin, spec.penal, nelx, nely)
        dc_tile = filters.grid_to_tile_sum(dc_el, nelx, nely, tx, ty)
        dH = filters.heaviside_derivative(xt, spec.beta, eta)
        dF += w[k] * filters.density_filter_adjoint(dH * dc_tile, tx, ty, spec.rmin)
        count = filters.grid_to_tile_sum(np.ones(nelx * nely), nelx, nely, tx, ty)
        dg += filters.density_filter_adjoint(dH * count, tx, ty, spec.rmin) / (m * nelx * nely * spec.volfrac)
    g = volume_constraint(xbars, nelx, nely, tx, ty, spec.volfrac)
    return F, c, g, dF, dg


def oc_update(spec, x_tile, dF, dg, move=0.2):
    """Optimality-criteria update with bisection on the multiplier (reading R11)."""
    nelx, nely, tx, ty = spec.nelx, spec.nely, spec.tile_x, spec.tile_y
    lo = np.maximum(0.0, x_tile - move)
    hi = np.minimum(1.0, x_tile + move)
    ratio = np.maximum(0.0, -dF) / np.maximum(dg, 1e-30)
    l1, l2 = 0.0, 1e9
    x_new = x_tile.copy()
    while (l2 - l1) / (l1 + l2) > 1e-3:
        lmid = 0.5 * (l1 + l2)
        x_new = np.clip(x_tile * np.sqrt(ratio / lmid), lo, hi)
        _, xbars = filters.physical_tiles(x_new, tx, ty, spec.rmin, spec.beta, spec.etas)
        if volume_constraint(xbars, nelx, nely, tx, ty, spec.volfrac) > 0.0:
            l1 = lmid
        else:
            l2 = lmid
    return x_new
