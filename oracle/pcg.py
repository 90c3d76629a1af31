"""ORACLE (test infrastructure only) -- preconditioned conjugate gradients.

PAPER.md §2.4.2 (line 146): "The linear elasticity problem, as well as the
preconditioner, is symmetric and positive definite and, hence, the preconditioned
conjugate gradient (PCG) method could be used."  The BASELINE north star fixes PCG; the
textbook PCG recurrence is written out below.

Reading R9: stop at the first iteration k with ||r_k||_2 <= tol * ||f||_2 (true
recursively-updated residual, 2-norm, relative to the load); the iteration count is the
number of operator applications A p performed; x0 = 0.
"""
from __future__ import annotations

import numpy as np


def pcg(apply_A, f, apply_M, tol=1e-8, max_it=1000, x0=None):
    """Returns (x, iterations, residual-norm history)."""
    x = np.zeros_like(f) if x0 is None else x0.copy()
    r = f - apply_A(x)
    fn = np.linalg.norm(f)
    hist = [np.linalg.norm(r)]
    if fn == 0.0 or hist[0] <= tol * fn:
        return x, 0, hist
    z = apply_M(r)
    p = z.copy()
    rz = r @ z
    for it in range(1, max_it + 1):
        q = apply_A(p)
        alpha = rz / (p @ q)
        x = x + alpha * p
        r = r - alpha * q
        hist.append(np.linalg.norm(r))
        if hist[-1] <= tol * fn:
            return x, it, hist
        z = apply_M(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, max_it, hist
