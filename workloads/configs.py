"""The five BASELINE.json configurations (plus small test variants).

Geometry/input conventions: SURVEY.md §8(c)-D13.  Element (i, j[, l]) is
centred at (i*p, j*p, l*p); vectors are X = (re + 1j*im).T with
re, im = default_rng(seed).standard_normal((nrhs, N)) drawn in that order.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .meshes import Mesh, cube_array


@dataclass(frozen=True)
class Config:
    name: str
    shape: tuple          # (nx, ny) planar or (nx, ny, nz) volumetric element counts
    period: float         # element period in wavelengths
    side: float | None    # cube side (None -> drawn per element, C3)
    n_per_face: int | None
    h: float
    M: int
    near_radius: float
    nrhs: int = 1
    k: float = 2.0 * math.pi
    side_seed: int | None = None
    side_range: tuple = (0.3, 0.5)
    cell: float = 0.05     # target square size for drawn sides (C3)
    notes: str = ""
    extra: dict = field(default_factory=dict)


CONFIGS = {
    # configs[0]: 2x2, 0.4 cubes, 4x4/face, h=0.1, M=2, r=0.3, 1 vector
    "c1": Config("c1", (2, 2), 0.5, 0.4, 4, 0.1, 2, 0.3, nrhs=1),
    # configs[1]: 10x10, 0.4 cubes, 8x8/face, h=0.05, M=2, r=0.2, 16 vectors
    "c2": Config("c2", (10, 10), 0.5, 0.4, 8, 0.05, 2, 0.2, nrhs=16),
    # configs[2]: 20x20 dissimilar, sides U[0.3,0.5] seed 1, ceil(s/0.05)^2/face
    "c3": Config("c3", (20, 20), 0.6, None, None, 0.05, 3, 0.2, nrhs=1, side_seed=1),
    # configs[3]: 32x32, 0.5 cubes, 10x10/face, h=0.05, M=3, r=0.2, plane wave + GMRES(50)
    "c4": Config("c4", (32, 32), 0.6, 0.5, 10, 0.05, 3, 0.2, nrhs=1),
    # configs[4]: 12x12x12 stack, 0.4 cubes, 6x6/face, h=0.05, M=2, r=0.2
    "c5": Config("c5", (12, 12, 12), 0.5, 0.4, 6, 0.05, 2, 0.2, nrhs=1),
    # --- small parity cases (not BASELINE configs): several tiles + ragged tails
    # 3x2 array, odd counts, M=3 (even stencil), h=0.1
    "t_m3": Config("t_m3", (3, 2), 0.5, 0.4, 4, 0.1, 3, 0.25, nrhs=1),
    # 2x2 of lambda/20 meshed cubes with configs-2..5 AIM parameters
    "t_fine_m2": Config("t_fine_m2", (2, 2), 0.5, 0.4, 8, 0.05, 2, 0.2, nrhs=1),
    "t_fine_m3": Config("t_fine_m3", (2, 2), 0.5, 0.4, 8, 0.05, 3, 0.2, nrhs=1),
    # dissimilar 3x3 (C3-like irregular occupancy), M=3
    "t_dissim": Config("t_dissim", (3, 3), 0.6, None, None, 0.05, 3, 0.2, nrhs=1, side_seed=1),
    # volumetric 2x2x2 (C5-like)
    "t_vol": Config("t_vol", (2, 2, 2), 0.5, 0.4, 4, 0.1, 2, 0.3, nrhs=1),
    # single cube, several RHS
    "t_one": Config("t_one", (1, 1), 0.5, 0.4, 3, 0.1, 2, 0.3, nrhs=3),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]


def element_layout(cfg: Config):
    """Element centres, sides and per-face subdivisions in element order."""
    dims = cfg.shape
    idx = np.indices(dims).reshape(len(dims), -1).T  # lexicographic, last axis fastest
    centers = np.zeros((idx.shape[0], 3))
    centers[:, : len(dims)] = idx * cfg.period
    if cfg.side is None:
        sides = np.random.default_rng(cfg.side_seed).uniform(
            cfg.side_range[0], cfg.side_range[1], dims).reshape(-1)
        ns = np.array([int(math.ceil(s / cfg.cell)) for s in sides])
    else:
        sides = np.full(idx.shape[0], cfg.side)
        ns = np.full(idx.shape[0], cfg.n_per_face)
    return centers, sides, ns


def make_mesh(cfg: Config | str) -> Mesh:
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    centers, sides, ns = element_layout(cfg)
    return cube_array(centers, sides, ns)


def make_vectors(n: int, nrhs: int = 1, seed: int = 0) -> np.ndarray:
    """[N][nrhs] complex128 with Re, Im iid N(0,1) (D13)."""
    g = np.random.default_rng(seed)
    re = g.standard_normal((nrhs, n))
    im = g.standard_normal((nrhs, n))
    return np.ascontiguousarray((re + 1j * im).T)
