"""ORACLE (test infrastructure only) -- one robust design evaluation, end to end.

PAPER.md §5.3 (lines 397-399): one spectral basis, built for the dilated realisation, is
re-used for the solves of all realisations ("the representative design is selected to
be the dilated one").  Each realisation has its own operator K(xbar_eta) and hence its own
Galerkin coarse matrix K_c = R_c K R_c^T (Eq. 10).
"""
from __future__ import annotations

import numpy as np

from . import fem, filters, msfem, pcg


def element_moduli(spec, x_tile):
    """Filter -> project per eta -> tile -> SIMP (§4.3, Eq. 16, Eq. 5)."""
    xt, xbars = filters.physical_tiles(x_tile, spec.tile_x, spec.tile_y, spec.rmin,
                                       spec.beta, spec.etas)
    xb_el = [filters.tile_to_grid(xb, spec.nelx, spec.nely, spec.tile_x, spec.tile_y)
             for xb in xbars]
    E_el = [fem.simp_modulus(x, spec.E0, spec.Emin, spec.penal) for x in xb_el]
    return xt, xbars, xb_el, E_el


def solve(spec, x_tile, fixed, f, tol=None, max_it=2000, smoother_only=False):
    tol = spec.tol if tol is None else tol
    K0 = fem.element_stiffness(spec.nu)
    xt, xbars, xb_el, E_el = element_moduli(spec, x_tile)
    R, eigvals = msfem.build_coarse_basis(spec.nelx, spec.nely, spec.cx, spec.cy,
                                          spec.n_modes, E_el[spec.dilated], K0, fixed,
                                          spec.lam_threshold)
    groups = msfem.gs_groups(spec.nelx, spec.nely, fixed)
    out = dict(K0=K0, xt=xt, xbars=xbars, E_el=E_el, R=R, eigvals=eigvals, us=[],
               iters=[], comps=[], hist=[], A=[], M=[])
    for k in range(len(spec.etas)):
        A = fem.constrained_operator(fem.assemble(spec.nelx, spec.nely, E_el[k], K0), fixed)
        M = msfem.TwoLevelPreconditioner(A, R, groups, fixed)
        if smoother_only:
            def Mfun(r, A=A):
                z = msfem.symmetric_gauss_seidel(A, np.zeros_like(r), r, groups)
                z[fixed != 0] = 0.0
                return z
        else:
            Mfun = M
        u, it, hist = pcg.pcg(lambda v, A=A: A @ v, f, Mfun, tol=tol, max_it=max_it)
        out["us"].append(u)
        out["iters"].append(it)
        out["comps"].append(fem.compliance(f, u))
        out["hist"].append(hist)
        out["A"].append(A)
        out["M"].append(M)
    return out
