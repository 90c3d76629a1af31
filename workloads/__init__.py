"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: only problem descriptors (grid sizes,
coarse-cell sizes, material constants), Dirichlet masks, load vectors and seeded random
design tiles.  Both sides (``oracle/`` and the CUDA path) consume what it produces; neither
side's numerics live here.

Conventions:
  * nodes (ix, iy), ix in [0, nelx], iy in [0, nely]; node id = ix*(nely+1) + iy (y fastest)
  * DOF id = 2*node + c, c = 0 (x) / 1 (y)
  * element (ex, ey), id = ex*nely + ey
  * design tile (tile_x, tile_y), id = tx*tile_y + ty; element (ex, ey) is controlled by tile
    variable ((ex % tile_x), (ey % tile_y))  -- PAPER.md §4.1 (lines 236-237): "the same design
    variable controls the relative density of several fine-scale elements".
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class ProblemSpec:
    name: str
    nelx: int
    nely: int
    cx: int                      # fine elements per coarse cell along x
    cy: int                      # fine elements per coarse cell along y
    n_modes: int                 # spectral eigenfunctions per agglomerate (cap)
    tile_x: int                  # design tile (periodic microstructure) size along x
    tile_y: int
    bc: str                      # 'cantilever' | 'mbb'
    design: str                  # 'iid' | 'binary'
    E0: float = 1.0
    Emin: float = 1e-9
    penal: float = 3.0
    nu: float = 0.3
    rmin: float = 0.0            # density filter radius in elements; < 1 -> identity filter
    beta: float = 0.0            # Heaviside sharpness; <= 0 -> identity projection
    etas: tuple = (0.5,)         # projection thresholds, one realisation each
    dilated: int = 0             # index into etas of the realisation that builds the basis
    volfrac: float = 0.5
    solid_fraction: float = 0.4  # for design == 'binary'
    seed: int = 0
    tol: float = 1e-8
    kappa: float = 1.0
    lam_threshold: float = float("inf")  # lambda_Omega; inf -> exactly n_modes per agglomerate

    @property
    def n_nodes(self) -> int:
        return (self.nelx + 1) * (self.nely + 1)

    @property
    def n_dof(self) -> int:
        return 2 * self.n_nodes

    @property
    def n_el(self) -> int:
        return self.nelx * self.nely

    @property
    def n_rhs(self) -> int:
        return len(self.etas)

    def replace(self, **kw) -> "ProblemSpec":
        return dataclasses.replace(self, **kw)


def node_id(spec: ProblemSpec, ix, iy):
    return np.asarray(ix) * (spec.nely + 1) + np.asarray(iy)


def fixed_mask(spec: ProblemSpec) -> np.ndarray:
    """uint8[n_dof]: 1 where the displacement is prescribed zero."""
    m = np.zeros(spec.n_dof, dtype=np.uint8)
    iy = np.arange(spec.nely + 1)
    if spec.bc == "cantilever":            # left edge clamped (both components)
        n = node_id(spec, 0, iy)
        m[2 * n] = 1
        m[2 * n + 1] = 1
    elif spec.bc == "mbb":                 # MBB half-beam: symmetry rollers + bottom-right support
        n = node_id(spec, 0, iy)
        m[2 * n] = 1
        m[2 * node_id(spec, spec.nelx, 0) + 1] = 1
    else:
        raise ValueError(f"unknown bc {spec.bc!r}")
    return m


def load_vector(spec: ProblemSpec) -> np.ndarray:
    """float64[n_dof]: unit point load (negative y)."""
    f = np.zeros(spec.n_dof, dtype=np.float64)
    if spec.bc == "cantilever":            # mid right edge
        f[2 * node_id(spec, spec.nelx, spec.nely // 2) + 1] = -1.0
    elif spec.bc == "mbb":                 # top-left corner
        f[2 * node_id(spec, 0, spec.nely) + 1] = -1.0
    return f


def design_tile(spec: ProblemSpec, seed: int | None = None) -> np.ndarray:
    """float64[tile_x*tile_y] seeded design variables on the unique tile."""
    rng = np.random.Generator(np.random.PCG64(spec.seed if seed is None else seed))
    n = spec.tile_x * spec.tile_y
    if spec.design == "iid":
        return rng.uniform(0.0, 1.0, size=n)
    if spec.design == "binary":
        return _connected_binary_cell(spec.tile_x, spec.tile_y, spec.solid_fraction, rng)
    if spec.design == "solid":   # homogeneous material (edge case: no contrast at all)
        return np.ones(n)
    raise ValueError(f"unknown design {spec.design!r}")


def _connected_binary_cell(tx: int, ty: int, frac: float, rng) -> np.ndarray:
    """Seeded 0/1 periodic cell with solid fraction ~frac whose solid is one connected
    (periodically tiled) phase: a frame of bars on the cell's left/bottom edges plus the
    super-level set of a smooth random periodic field, keeping only the solid components
    connected to the frame.  (Floating islands would each add 3 rigid modes per
    agglomerate; the BASELINE contrast sweep wants a connected microstructure.)"""
    X, Y = np.meshgrid(np.arange(tx) / tx, np.arange(ty) / ty, indexing="ij")
    field = np.zeros((tx, ty))
    for _ in range(12):
        kx, ky = rng.integers(-3, 4, size=2)
        ph = rng.uniform(0, 2 * np.pi)
        field += rng.standard_normal() * np.cos(2 * np.pi * (kx * X + ky * Y) + ph)
    w = max(1, min(tx, ty) // 10)
    frame = np.zeros((tx, ty), dtype=bool)
    frame[:w, :] = True
    frame[:, :w] = True

    def connected(solid):
        seen = frame & solid
        stack = list(zip(*np.nonzero(seen)))
        while stack:
            i, j = stack.pop()
            for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                a, b = (i + di) % tx, (j + dj) % ty
                if solid[a, b] and not seen[a, b]:
                    seen[a, b] = True
                    stack.append((a, b))
        return seen

    best = None
    for q in np.linspace(0.0, 1.0, 101):
        thr = np.quantile(field, q)
        cell = connected(frame | (field > thr))
        err = abs(cell.mean() - frac)
        if best is None or err < best[0]:
            best = (err, cell)
    return best[1].astype(np.float64).ravel()


def random_vectors(n: int, k: int, seed: int) -> np.ndarray:
    """float64[k, n] seeded standard normals (test probes)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal((k, n))


# ---------------------------------------------------------------------------------------
# BASELINE.json configs.  configs[0] is the small case the oracle finishes in seconds,
# configs[1] is the bench workload (fits one B200), the rest are parity / property cases.
# ---------------------------------------------------------------------------------------
CONFIGS = {
    # configs[0]: cantilever 96x48, iid densities, 8x8 coarse cells, 4 modes, single solve
    "c0_cantilever_96x48": ProblemSpec(
        name="c0_cantilever_96x48", nelx=96, nely=48, cx=8, cy=8, n_modes=4,
        tile_x=96, tile_y=48, bc="cantilever", design="iid", Emin=1e-9, penal=3.0,
        etas=(0.5,), dilated=0, tol=1e-8, seed=1),
    # configs[1]: MBB 1024x512, 32x32 periodic random cells, filter 2.5, beta 8, 3 robust RHS
    "c1_mbb_1024x512": ProblemSpec(
        name="c1_mbb_1024x512", nelx=1024, nely=512, cx=16, cy=16, n_modes=4,
        tile_x=32, tile_y=32, bc="mbb", design="iid", Emin=1e-9, penal=3.0,
        rmin=2.5, beta=8.0, etas=(0.7, 0.5, 0.3), dilated=2, tol=1e-8, seed=2),
    # configs[2]: cantilever 2048x1024, layered (x-periodic 64, constant in y), 6 modes
    "c2_cantilever_2048x1024": ProblemSpec(
        name="c2_cantilever_2048x1024", nelx=2048, nely=1024, cx=16, cy=16, n_modes=6,
        tile_x=64, tile_y=1, bc="cantilever", design="iid", Emin=1e-9, penal=3.0,
        rmin=2.5, beta=8.0, etas=(0.7, 0.5, 0.3), dilated=2, volfrac=0.5, tol=1e-8, seed=3),
    # configs[3]: contrast sweep 2048x2048 binary periodic 32x32 cells (solid 0.4); the
    # paper's lambda_Omega selection with a 16-mode cap (reading R5):
    # a fixed 4 modes is not contrast-independent for a binary microstructure
    "c3_square_2048": ProblemSpec(
        name="c3_square_2048", nelx=2048, nely=2048, cx=16, cy=16, n_modes=16,
        tile_x=32, tile_y=32, bc="cantilever", design="binary", Emin=1e-9, penal=3.0,
        etas=(0.5,), dilated=0, tol=1e-8, seed=4, lam_threshold=5e-3),
    # configs[4]: MBB 5120x2560 (~26.2M DOF), 40x40 cells, 20x20 coarse, 3 robust RHS
    "c4_mbb_5120x2560": ProblemSpec(
        name="c4_mbb_5120x2560", nelx=5120, nely=2560, cx=20, cy=20, n_modes=4,
        tile_x=40, tile_y=40, bc="mbb", design="iid", Emin=1e-9, penal=3.0,
        rmin=2.5, beta=8.0, etas=(0.7, 0.5, 0.3), dilated=2, tol=1e-8, seed=5),
}


def small_spec(nelx=16, nely=8, cx=4, cy=4, n_modes=4, bc="cantilever", tile=None,
               design="iid", rmin=0.0, beta=0.0, etas=(0.5,), dilated=0, Emin=1e-9,
               seed=7, **kw) -> ProblemSpec:
    """A small problem the oracle solves in well under a second."""
    tx, ty = tile if tile is not None else (nelx, nely)
    return ProblemSpec(name=f"small_{nelx}x{nely}", nelx=nelx, nely=nely, cx=cx, cy=cy,
                       n_modes=n_modes, tile_x=tx, tile_y=ty, bc=bc, design=design,
                       rmin=rmin, beta=beta, etas=tuple(etas), dilated=dilated, Emin=Emin,
                       seed=seed, **kw)
