"""Synthetic DEMs for the D8 flow-direction stencil.

The paper times flow direction on two unnamed DEMs of 339 x 225 and 14786 x 10086 points;
neither is available, so these seeded rasters of the same sizes stand in for them: the 16 random-phase
sinusoids of cfg2/cfg4 (stream 1 draws), each evaluated in the separable form
sin(kx x) cos(ky y + phi) + cos(kx x) sin(ky y + phi) so that 150 M points generate in seconds, rescaled
to 300 m of relief above 10 m, quantised to 1 cm (real DEMs are
quantised, which makes ties between neighbours common), with a no-data disc (value -9999, which the
paper's user function skips through its `nghb[i] > 0` test) covering ~5 % of the raster.
"""
from __future__ import annotations

import numpy as np

from .configs import _centres, _sinusoid_params

DEM_SIZES = {"dem_small": (339, 225), "dem_large": (14786, 10086)}
NODATA = -9999.0


def make_dem(nx: int, ny: int, dtype=np.float64, quantum: float = 0.01, nodata: bool = True) -> np.ndarray:
    lam, theta, phi = _sinusoid_params()
    x = _centres(nx, 1.0)
    y = _centres(ny, 1.0)
    z = np.zeros((ny, nx), dtype=np.float64)
    for k in range(16):
        kx, ky = 2.0 * np.pi * np.cos(theta[k]) / lam[k], 2.0 * np.pi * np.sin(theta[k]) / lam[k]
        z += np.outer(np.cos(ky * y + phi[k]), np.sin(kx * x))
        z += np.outer(np.sin(ky * y + phi[k]), np.cos(kx * x))
    zmin, zmax = z.min(), z.max()
    z -= zmin
    z *= 300.0 / (zmax - zmin)
    z += 10.0
    if quantum:
        np.round(z / quantum, out=z)
        z *= quantum
    if nodata:
        r = 0.13 * min(nx, ny)
        y, x = np.ogrid[:ny, :nx]
        disc = (x - 0.7 * nx) ** 2 + (y - 0.3 * ny) ** 2 < r * r
        z[disc] = NODATA
    return np.ascontiguousarray(z.astype(dtype, copy=False))


def make_named(name: str, dtype=np.float64) -> np.ndarray:
    nx, ny = DEM_SIZES[name]
    return make_dem(nx, ny, dtype=dtype)
