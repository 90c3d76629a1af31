"""Pins of oracle/filters.py: Eq. 16 special values, brute-force periodic filter, adjoints."""
import numpy as np
import pytest

from oracle import filters


@pytest.mark.parametrize("beta", [1.0, 8.0, 64.0])
@pytest.mark.parametrize("eta", [0.3, 0.5, 0.7])
def test_heaviside_endpoints_and_monotone(beta, eta):
    x = np.linspace(0, 1, 101)
    h = filters.heaviside(x, beta, eta)
    assert abs(h[0]) < 1e-15 and abs(h[-1] - 1) < 1e-15
    assert np.all(np.diff(h) >= 0) and (beta > 8 or np.all(np.diff(h) > 0))
    assert np.all((h >= -1e-15) & (h <= 1 + 1e-15))


def test_heaviside_symmetry_point():
    for beta in (1.0, 8.0, 100.0):
        assert abs(filters.heaviside(np.array(0.5), beta, 0.5) - 0.5) < 1e-15


def test_heaviside_derivative_fd_and_peak():
    rng = np.random.default_rng(0)
    x = rng.uniform(0.05, 0.95, 20)
    for beta, eta in ((8.0, 0.3), (16.0, 0.5), (32.0, 0.7)):
        h = 1e-6
        fd = (filters.heaviside(x + h, beta, eta) - filters.heaviside(x - h, beta, eta)) / (2 * h)
        an = filters.heaviside_derivative(x, beta, eta)
        assert np.abs(fd - an).max() < 1e-7 * max(1.0, np.abs(an).max())
        grid = np.linspace(0, 1, 10001)
        assert abs(grid[np.argmax(filters.heaviside_derivative(grid, beta, eta))] - eta) < 1e-4


def test_projection_identity_when_beta_nonpositive():
    x = np.random.default_rng(1).uniform(size=10)
    assert np.array_equal(filters.heaviside(x, 0.0, 0.5), x)
    assert np.array_equal(filters.heaviside_derivative(x, 0.0, 0.5), np.ones(10))


def test_projection_eta_ordering():
    """eta1 < eta2 -> xbar(eta1) >= xbar(eta2): dilated embeds eroded."""
    x = np.linspace(0, 1, 501)
    a, b, c = (filters.heaviside(x, 8.0, e) for e in (0.3, 0.5, 0.7))
    assert np.all(a >= b - 1e-15) and np.all(b >= c - 1e-15)


def brute_force_filter(x, tx, ty, rmin):
    X = x.reshape(tx, ty)
    out = np.zeros_like(X)
    r = int(np.ceil(rmin))
    for i in range(tx):
        for j in range(ty):
            num = den = 0.0
            for dx in range(-r, r + 1):
                for dy in range(-r, r + 1):
                    w = max(0.0, rmin - np.sqrt(dx * dx + dy * dy))
                    num += w * X[(i + dx) % tx, (j + dy) % ty]
                    den += w
            out[i, j] = num / den
    return out.ravel()


@pytest.mark.parametrize("tx,ty,rmin", [(5, 5, 2.0), (8, 6, 2.5), (7, 3, 1.5), (6, 1, 2.5)])
def test_filter_equals_brute_force_toroidal(tx, ty, rmin):
    x = np.random.default_rng(2).uniform(size=tx * ty)
    assert np.abs(filters.density_filter(x, tx, ty, rmin) - brute_force_filter(x, tx, ty, rmin)).max() < 1e-14


def test_filter_spike_and_uniform_and_identity():
    tx = ty = 5
    x = np.zeros(25); x[12] = 1.0
    out = filters.density_filter(x, tx, ty, 2.0).reshape(5, 5)
    w = {(0, 0): 2.0, (1, 0): 1.0, (1, 1): 2.0 - np.sqrt(2.0)}
    tot = w[(0, 0)] + 4 * w[(1, 0)] + 4 * w[(1, 1)]
    assert abs(out[2, 2] - 2.0 / tot) < 1e-15
    assert abs(out[3, 3] - w[(1, 1)] / tot) < 1e-15
    assert abs(out[0, 0]) < 1e-15
    u = np.full(30, 0.37)
    assert np.abs(filters.density_filter(u, 6, 5, 2.5) - 0.37).max() < 1e-15
    y = np.random.default_rng(3).uniform(size=30)
    assert np.array_equal(filters.density_filter(y, 6, 5, 0.5), y)


def test_filter_translation_equivariance_and_bounds():
    tx, ty = 8, 6
    x = np.random.default_rng(4).uniform(size=tx * ty)
    X = x.reshape(tx, ty)
    f1 = filters.density_filter(np.roll(X, 3, axis=0).ravel(), tx, ty, 2.5).reshape(tx, ty)
    f2 = np.roll(filters.density_filter(x, tx, ty, 2.5).reshape(tx, ty), 3, axis=0)
    assert np.abs(f1 - f2).max() < 1e-15
    fx = filters.density_filter(x, tx, ty, 2.5)
    assert fx.min() >= x.min() - 1e-15 and fx.max() <= x.max() + 1e-15


def test_filter_adjoint_identity():
    tx, ty = 7, 5
    rng = np.random.default_rng(5)
    x, y = rng.standard_normal(tx * ty), rng.standard_normal(tx * ty)
    lhs = filters.density_filter(x, tx, ty, 2.5) @ y
    rhs = x @ filters.density_filter_adjoint(y, tx, ty, 2.5)
    assert abs(lhs - rhs) < 1e-13 * abs(lhs)


def test_tiling_maps_adjoint_and_periodic():
    nelx, nely, tx, ty = 12, 8, 4, 4
    rng = np.random.default_rng(6)
    v, w = rng.standard_normal(tx * ty), rng.standard_normal(nelx * nely)
    g = filters.tile_to_grid(v, nelx, nely, tx, ty)
    assert abs(g @ w - v @ filters.grid_to_tile_sum(w, nelx, nely, tx, ty)) < 1e-12
    G = g.reshape(nelx, nely)
    assert np.array_equal(G[:4, :4], G[4:8, 4:8]) and np.array_equal(G[:4], G[8:12])
    assert np.allclose(filters.grid_to_tile_sum(np.ones(nelx * nely), nelx, nely, tx, ty), 6.0)
