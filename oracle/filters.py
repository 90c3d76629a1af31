"""ORACLE (test infrastructure only) -- density filter, Heaviside projection, tiling.

PAPER.md §4.3 (lines 259-275): design variables are filtered by the standard
neighbourhood density filter and then projected with the smoothed Heaviside Eq. 16
(line 263); for a single periodic microstructure "periodicity is introduced by applying
the standard filter on a 3x3 block of the microstructural design" (line 275).
PAPER.md §4.1 (line 236): the same design variable controls several fine elements
(tiling map); the total sensitivity sums the local sensitivities of all controlled
elements.

Readings: R3 cone weights w(d) = max(0, rmin - |d|) on integer element-centre offsets,
normalised by their sum; the 3x3-block periodic filter is the toroidal (wrap-around)
filter of the tile (identical whenever rmin <= tile size; the wrap form is used for any
size).  rmin < 1 gives the identity filter.  R4 beta <= 0 means "no projection"
(identity), used for configs whose physical density is given directly.
"""
from __future__ import annotations

import numpy as np


def filter_offsets(rmin: float):
    """Integer offsets (dx, dy) with positive cone weight max(0, rmin - |d|)."""
    r = int(np.ceil(rmin)) - 1 if rmin >= 1.0 else 0
    out = []
    for dx in range(-r, r + 1):
        for dy in range(-r, r + 1):
            w = max(0.0, rmin - np.hypot(dx, dy))
            if w > 0.0:
                out.append((dx, dy, w))
    if not out:
        out = [(0, 0, 1.0)]
    return out


def density_filter(x_tile: np.ndarray, tile_x: int, tile_y: int, rmin: float) -> np.ndarray:
    """x~_t = sum_d w(d) x_{(t+d) mod tile} / sum_d w(d)   (§4.3, line 261/275)."""
    X = x_tile.reshape(tile_x, tile_y)
    acc = np.zeros_like(X)
    wsum = 0.0
    for dx, dy, w in filter_offsets(rmin):
        acc += w * np.roll(np.roll(X, -dx, axis=0), -dy, axis=1)
        wsum += w
    return (acc / wsum).ravel()


def density_filter_adjoint(g_tile: np.ndarray, tile_x: int, tile_y: int, rmin: float) -> np.ndarray:
    """W^T g for the filter above (chain rule)."""
    G = g_tile.reshape(tile_x, tile_y)
    acc = np.zeros_like(G)
    wsum = 0.0
    for dx, dy, w in filter_offsets(rmin):
        acc += w * np.roll(np.roll(G, dx, axis=0), dy, axis=1)
        wsum += w
    return (acc / wsum).ravel()


def heaviside(xt: np.ndarray, beta: float, eta: float) -> np.ndarray:
    """PAPER.md Eq. 16 (line 263):
    xbar = (tanh(beta eta) + tanh(beta (x~ - eta))) / (tanh(beta eta) + tanh(beta (1 - eta)))."""
    if beta <= 0.0:
        return np.array(xt, dtype=np.float64, copy=True)
    num = np.tanh(beta * eta) + np.tanh(beta * (xt - eta))
    den = np.tanh(beta * eta) + np.tanh(beta * (1.0 - eta))
    return num / den


def heaviside_derivative(xt: np.ndarray, beta: float, eta: float) -> np.ndarray:
    """d xbar / d x~ of Eq. 16 (chain rule)."""
    if beta <= 0.0:
        return np.ones_like(xt)
    den = np.tanh(beta * eta) + np.tanh(beta * (1.0 - eta))
    return beta * (1.0 - np.tanh(beta * (xt - eta)) ** 2) / den


def tile_to_grid(v_tile: np.ndarray, nelx: int, nely: int, tile_x: int, tile_y: int) -> np.ndarray:
    """Element field from a tile field (§4.1 line 236 tiling map)."""
    ex, ey = np.meshgrid(np.arange(nelx), np.arange(nely), indexing="ij")
    return v_tile[((ex % tile_x) * tile_y + (ey % tile_y)).ravel()]


def grid_to_tile_sum(v_el: np.ndarray, nelx: int, nely: int, tile_x: int, tile_y: int) -> np.ndarray:
    """Sum of element values over all elements controlled by each tile variable
    ("summing up local sensitivities of all fine-scale elements")."""
    ex, ey = np.meshgrid(np.arange(nelx), np.arange(nely), indexing="ij")
    t = ((ex % tile_x) * tile_y + (ey % tile_y)).ravel()
    return np.bincount(t, weights=v_el, minlength=tile_x * tile_y)


def physical_tiles(x_tile, tile_x, tile_y, rmin, beta, etas):
    """Filtered tile and one projected tile per threshold eta (§4.4:
    "several projections using different threshold values")."""
    xt = density_filter(x_tile, tile_x, tile_y, rmin)
    return xt, [heaviside(xt, beta, eta) for eta in etas]
