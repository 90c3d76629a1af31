"""GPU checks on BASELINE configs[3], the contrast-independence sweep (2048 x 2048 elements,
binary periodic cell, lambda_Omega threshold mode with up to 16 modes per agglomerate, E_min in
{1e-3, 1e-6, 1e-9}; section 3.1, l.132 the threshold).  It is the one config
that takes the 16-mode paths at full size: four 16-column groups in the restriction /
prolongation kernels, 64 x 64 Galerkin cell matrices, and the long fronts of the nested
dissection (several row stages per CTA in the coarse solve).  The oracle cannot assemble or
solve it, so, as in test_gpu_fullsize_large.py: the operator row by row at sampled nodes, the
kept local spectra of sampled agglomerates against the oracle's dense eigensolver, the coarse
solve through the residual of the gathered K_c, preconditioner symmetry, the PCG solution
through its true residual; and the paper's claim itself, iteration counts that stay flat from
E_min = 1e-6 to 1e-9."""
import numpy as np
import pytest

import workloads as W
from oracle import fem, msfem, problem

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():
    pytest.skip("no GPU", allow_module_level=True)

from paper_1411_3923_b200 import Msfem, build  # noqa: E402
from test_gpu_fullsize_large import coarse_residual_check, host, operator_rows  # noqa: E402

build.build()
DEV = torch.device("cuda")
NAME = "c3_square_2048"


def context(emin):
    spec = W.CONFIGS[NAME].replace(Emin=emin)
    x = W.design_tile(spec)
    m = Msfem.from_spec(spec)
    m.filter_project(torch.as_tensor(x, device=DEV))
    m.build_coarse_basis()
    m.assemble_coarse()
    return spec, x, m


@pytest.fixture(scope="module")
def case():
    spec, x, m = context(1e-9)
    xt, xbars, xb_el, E = problem.element_moduli(spec, x)
    yield dict(spec=spec, m=m, x=x, E=E, fx=W.fixed_mask(spec), f=W.load_vector(spec),
               K0=fem.element_stiffness(spec.nu))
    m.close()
    torch.cuda.empty_cache()


def test_contrast_operator_sampled_rows(case):
    spec, m = case["spec"], case["m"]
    nny = spec.nely + 1
    v = W.random_vectors(spec.n_dof, 1, seed=5)[0]
    nodes = list(np.random.default_rng(7).choice(spec.n_dof // 2, 300, replace=False))
    nodes += [iy for iy in (0, nny // 2, nny - 1)] + [spec.nelx * nny + iy for iy in (0, nny - 1)]
    y = torch.empty(spec.n_dof, dtype=torch.float64, device=DEV)
    m.matvec(0, torch.as_tensor(v, device=DEV), y)
    Y = host(y).reshape(-1, 2)[nodes]
    ref = operator_rows(spec, case["E"][0], case["K0"], case["fx"], v, nodes)
    assert np.abs(Y - ref).max() <= 1e-13 * np.abs(ref).max()


def test_contrast_kept_spectra_below_threshold(case):
    """Threshold mode (reading R5): exactly the eigenvalues below lambda_Omega are kept."""
    spec, m = case["spec"], case["m"]
    _, nk, lam = m.get_basis()
    ncx, ncy = spec.nelx // spec.cx, spec.nely // spec.cy
    for I, J in [(0, 0), (ncx, ncy // 2), (ncx // 2, ncy // 3)]:
        Kl, D, *_ = msfem.local_problem(I, J, spec.nelx, spec.nely, spec.cx, spec.cy,
                                        case["E"][spec.dilated], case["K0"], case["fx"])
        lo, _ = msfem.local_eigenpairs(Kl, D, spec.n_modes)
        agg = I * (ncy + 1) + J
        k = int(nk[agg])
        assert 3 <= k <= spec.n_modes
        assert k == min(spec.n_modes, int((lo < spec.lam_threshold).sum())), (I, J, k, lo)
        assert np.abs(lam[agg][:k] - lo[:k]).max() <= 1e-9 * max(1.0, np.abs(lo[:k]).max()), (I, J)


def test_contrast_coarse_solve_residual(case):
    """K_c c = b through the long fronts (k = 16: several row stages per CTA)."""
    coarse_residual_check(case["spec"], case["m"], (0,))


def test_contrast_preconditioner_symmetric(case):
    spec, m, fx = case["spec"], case["m"], case["fx"]
    V = W.random_vectors(spec.n_dof, 2, seed=13)
    V[:, fx == 1] = 0
    Z = []
    for v in V:
        z = torch.empty(spec.n_dof, dtype=torch.float64, device=DEV)
        m.precond_apply(0, torch.as_tensor(v, device=DEV), z)
        Z.append(host(z))
    assert Z[0] @ V[0] > 0 and Z[1] @ V[1] > 0
    a, b = Z[0] @ V[1], Z[1] @ V[0]
    assert abs(a - b) <= 1e-9 * max(abs(a), abs(b))


def test_contrast_pcg_true_residual(case):
    spec, m, f = case["spec"], case["m"], case["f"]
    u = torch.empty(spec.n_dof, dtype=torch.float64, device=DEV)
    its, comps, noconv = m.pcg_solve(tol=spec.tol, max_it=2000, u=u)
    assert not noconv and its[0] <= 80, its
    fd = torch.as_tensor(f, device=DEV)
    Ku = torch.empty_like(u)
    m.matvec(0, u, Ku)
    k_inf = 4 * spec.E0 * np.abs(case["K0"]).sum(axis=1).max()
    rn, un = float(torch.linalg.norm(fd - Ku)), float(torch.linalg.norm(u))
    assert rn <= 10 * spec.tol * float(torch.linalg.norm(fd)) + 10 * np.finfo(np.float64).eps * k_inf * un
    assert abs(comps[0] - float(fd @ u)) <= 1e-12 * abs(comps[0])


def test_contrast_iterations_flat(case):
    """the iteration count does not grow with the contrast.  E_min = 1e-9
    comes from the module's context, 1e-3 and 1e-6 from fresh ones."""
    its = {}
    its[1e-9] = case["m"].pcg_solve(tol=case["spec"].tol, max_it=2000)[0][0]
    for emin in (1e-3, 1e-6):
        spec, x, m = context(emin)
        its[emin] = m.pcg_solve(tol=spec.tol, max_it=2000)[0][0]
        m.close()
        del m
        torch.cuda.empty_cache()
    assert abs(its[1e-9] - its[1e-6]) <= 0.1 * its[1e-6] + 1, its
    assert its[1e-9] <= 1.6 * its[1e-3], its
