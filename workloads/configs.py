"""The five BASELINE.json workloads (cfg0..cfg4, zero-based) as concrete, seeded problem statements.

Recipes follow SURVEY.md §8d's table; every input is generated ONCE on the host and handed to both
the oracle and the CUDA path.  Each `make_cfgK(nx, ny)` also builds a geometrically scaled variant of
the same recipe (same physics, fewer cells) used for oracle-sized parity tests.

Conventions: cell (i, j) has centre x = (i + 1/2) dx, y = (j + 1/2) dy; arrays are row-major
(ny, nx) with x fastest; SI units (m, s); rain is stored in m/s (host conversion mm/h -> m/s is
(r / 1000) / 3600).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import rng

CONFIG_NAMES = ("cfg0", "cfg1", "cfg2", "cfg3", "cfg4")
SIDES = ("W", "E", "S", "N")
BC_TYPES = ("wall", "free", "periodic", "inflow")
FRICTION_LAWS = ("none", "manning", "strickler", "darcy_weisbach", "chezy")


def mm_per_h(r: float) -> float:
    return (r / 1000.0) / 3600.0


@dataclass
class GreenAmpt:
    Ks: float = 1e-6       # saturated hydraulic conductivity [m/s]
    hf: float = 0.1        # wetting-front capillary head [m]
    A: float = 1.0         # modified Green-Ampt offset (paper P:366, value not given; Q15)
    dtheta: float = 0.3    # theta_s - theta_i
    vinf0: float = 0.003   # initial infiltrated volume per area [m] (Q15: dtheta * 0.01 m)


@dataclass
class Inflow:
    k0: int                      # first boundary cell of the inflow segment
    k1: int                      # one past the last
    hydro_t: list                # hydrograph times [s] (piecewise linear, clamped at the ends)
    hydro_q: list                # discharge Q(t) [m^3/s] over the whole segment
    width: float = 0.0           # width Q is spread over [m] (0: the segment's own); strips of a
                                 # decomposed grid keep the global segment's width (paper_1307_4839_b200.sharded)


@dataclass
class SwofConfig:
    name: str
    nx: int
    ny: int
    dx: float
    dy: float
    g: float = 9.81
    cfl: float = 0.4
    dt_max: float = 1.0
    h_eps: float = 1e-12
    fric_law: str = "none"
    fric_coef: float = 0.0
    ga: Optional[GreenAmpt] = None
    rain_t: list = field(default_factory=list)     # piecewise-constant rain: R(t) = rate[k] for t in [t_k, t_k+1)
    rain_rate: list = field(default_factory=list)  # m/s
    bc: dict = field(default_factory=lambda: {s: "wall" for s in SIDES})
    inflow: dict = field(default_factory=dict)     # side -> Inflow
    # scheme variants; the defaults are the paper's recommended scheme
    flux: str = "hll"                              # "hll" | "rusanov"
    order: int = 2                                 # 2: MUSCL + Heun | 1: first order, explicit Euler
    cfl_mode: str = "cell"                         # "cell" (Q10) | "face": reconstructed values
    ga_form: str = "printed"                       # "printed" | "darcy": h_f + h_over (Q15)
    clamp_fail: float = 0.0                        # largest tolerated single clamp [m] (0: library default)
    dry_skip: bool = False                         # GPU: skip the stencil work of all-dry tiles (results unchanged)
    steps: Optional[int] = None                    # fixed step count (swof_step), or
    t_end: Optional[float] = None                  # run to t_end (swof_run)
    # inputs
    z: np.ndarray = None
    h: np.ndarray = None
    hu: np.ndarray = None
    hv: np.ndarray = None
    vinf: Optional[np.ndarray] = None
    fric_field: Optional[np.ndarray] = None        # per-cell friction coefficient (same law), or None

    @property
    def cells(self) -> int:
        return self.nx * self.ny

    def describe(self) -> dict:
        return {"workload": self.name, "nx": self.nx, "ny": self.ny, "dx": self.dx, "dy": self.dy,
                "fric_law": self.fric_law, "ga": self.ga is not None, "rain": bool(self.rain_rate),
                "bc": dict(self.bc), "steps": self.steps, "t_end": self.t_end}


def _centres(n: int, d: float) -> np.ndarray:
    return (np.arange(n, dtype=np.float64) + 0.5) * d


def _zeros(ny, nx):
    return np.zeros((ny, nx), dtype=np.float64)


# ----------------------------------------------------------------------------------------------
# cfg0: 64x64 lake at rest over a Gaussian bump with a Gaussian water hump, 4 walls, Manning 0.03
# ----------------------------------------------------------------------------------------------
def make_cfg0(nx: int = 64, ny: int = 64, steps: int = 200) -> SwofConfig:
    dx = dy = 1.0
    x = _centres(nx, dx)[None, :]
    y = _centres(ny, dy)[:, None]
    cx, cy = 32.0 * nx / 64.0, 32.0 * ny / 64.0
    hx, hy = 20.0 * nx / 64.0, 20.0 * ny / 64.0
    # (x-32)^2 + (y-32)^2 as two separately rounded squares: transpose-symmetric bit for bit
    z = 0.5 * np.exp(-(((x - cx) ** 2) + ((y - cy) ** 2)) / 50.0)
    h = np.maximum(0.0, 1.0 - z) + 0.1 * np.exp(-(((x - hx) ** 2) + ((y - hy) ** 2)) / 10.0)
    return SwofConfig(name="cfg0", nx=nx, ny=ny, dx=dx, dy=dy, fric_law="manning", fric_coef=0.03,
                      steps=steps, z=np.ascontiguousarray(z), h=np.ascontiguousarray(h),
                      hu=_zeros(ny, nx), hv=_zeros(ny, nx))


# ----------------------------------------------------------------------------------------------
# cfg1: 1024^2, dx 0.5 m, 1% slope down to the east, dry-bed dam break, Darcy-Weisbach f = 0.05
# ----------------------------------------------------------------------------------------------
def make_cfg1(nx: int = 1024, ny: int = 1024, steps: int = 2000) -> SwofConfig:
    dx = dy = 0.5
    Lx = nx * dx
    x = _centres(nx, dx)
    z = np.broadcast_to(0.01 * (Lx - x), (ny, nx)).copy()
    h = _zeros(ny, nx)
    h[:, : nx // 2] = 2.0            # h = 2 m for x < Lx/2 (256 m at full size)
    bc = {"W": "wall", "E": "free", "S": "wall", "N": "wall"}
    return SwofConfig(name="cfg1", nx=nx, ny=ny, dx=dx, dy=dy, fric_law="darcy_weisbach",
                      fric_coef=0.05, bc=bc, steps=steps, z=z, h=h, hu=_zeros(ny, nx), hv=_zeros(ny, nx))


# ----------------------------------------------------------------------------------------------
# sinusoid terrain generator shared by cfg2 and cfg4 (stream 1: lambda_k, theta_k, phi_k)
# ----------------------------------------------------------------------------------------------
def _sinusoid_params():
    u = rng.uniform(1, 48).reshape(16, 3)
    lam = 20.0 * (500.0 / 20.0) ** u[:, 0]        # log-uniform in [20, 500] m
    theta = 2.0 * np.pi * u[:, 1]
    phi = 2.0 * np.pi * u[:, 2]
    return lam, theta, phi


def _sinusoid_terrain(nx, ny, dx, dy, amp_total=5.0, rows_per_chunk=512):
    lam, theta, phi = _sinusoid_params()
    x = _centres(nx, dx)[None, :]
    z = np.empty((ny, nx), dtype=np.float64)
    a = amp_total / 16.0
    for j0 in range(0, ny, rows_per_chunk):
        j1 = min(ny, j0 + rows_per_chunk)
        y = _centres(ny, dy)[j0:j1, None]
        acc = np.zeros((j1 - j0, nx), dtype=np.float64)
        for k in range(16):
            acc += a * np.sin(2.0 * np.pi * (x * np.cos(theta[k]) + y * np.sin(theta[k])) / lam[k] + phi[k])
        z[j0:j1] = acc
    return z


# ----------------------------------------------------------------------------------------------
# cfg2: 2048^2 sinusoid terrain + 0.5% slope, dry, rain 50 mm/h for 600 s, Green-Ampt, to t = 900 s
# ----------------------------------------------------------------------------------------------
def make_cfg2(nx: int = 2048, ny: int = 2048, t_end: float = 900.0) -> SwofConfig:
    dx = dy = 1.0
    Lx = nx * dx
    z = _sinusoid_terrain(nx, ny, dx, dy) + 0.005 * (Lx - _centres(nx, dx))[None, :]
    bc = {"W": "wall", "E": "free", "S": "wall", "N": "wall"}
    return SwofConfig(name="cfg2", nx=nx, ny=ny, dx=dx, dy=dy, fric_law="manning", fric_coef=0.05,
                      ga=GreenAmpt(), rain_t=[0.0, 600.0], rain_rate=[mm_per_h(50.0), 0.0], bc=bc,
                      t_end=t_end, z=np.ascontiguousarray(z), h=_zeros(ny, nx), hu=_zeros(ny, nx),
                      hv=_zeros(ny, nx), vinf=np.full((ny, nx), GreenAmpt().vinf0))


# ----------------------------------------------------------------------------------------------
# cfg3: 4096^2, dx 2 m, diamond-square valley (stream 5) with a carved channel, inflow hydrograph
#       on the channel's west end, Manning n per cell ~ U[0.02, 0.08] (stream 4), rain + GA
# ----------------------------------------------------------------------------------------------
def diamond_square(n_pow2: int, roughness: float = 0.6, stream: int = 5) -> np.ndarray:
    """Classic diamond-square on a (2^k+1)^2 lattice; uniforms drawn in a fixed order from `stream`."""
    N = n_pow2 + 1
    a = np.zeros((N, N), dtype=np.float64)
    ctr = [0]

    def draw(shape):
        n = int(np.prod(shape))
        u = rng.uniform(stream, n, ctr[0]).reshape(shape)
        ctr[0] += n
        return 2.0 * u - 1.0

    amp = 1.0
    a[0::N - 1, 0::N - 1] = draw((2, 2)) * amp
    step = N - 1
    while step > 1:
        half = step // 2
        amp *= roughness
        # diamond step: square centres
        c = (a[0:-1:step, 0:-1:step] + a[0:-1:step, step::step] + a[step::step, 0:-1:step]
             + a[step::step, step::step]) * 0.25
        a[half::step, half::step] = c + amp * draw(c.shape)
        # square step: edge midpoints, average of the 3 or 4 lattice neighbours at distance `half`
        for (r0, c0) in ((0, half), (half, 0)):
            rows = np.arange(r0, N, step)
            cols = np.arange(c0, N, step)
            R, C = np.meshgrid(rows, cols, indexing="ij")
            s = np.zeros(R.shape)
            cnt = np.zeros(R.shape)
            for dr, dc in ((-half, 0), (half, 0), (0, -half), (0, half)):
                rr, cc = R + dr, C + dc
                ok = (rr >= 0) & (rr < N) & (cc >= 0) & (cc < N)
                s[ok] += a[rr[ok], cc[ok]]
                cnt[ok] += 1.0
            a[R, C] = s / cnt + amp * draw(R.shape)
        step = half
    return a


def make_cfg3(nx: int = 4096, ny: int = 4096, steps: int = 5000, channel_cells: Optional[int] = None) -> SwofConfig:
    dx = dy = 2.0
    Lx, Ly = nx * dx, ny * dy
    k = int(np.ceil(np.log2(max(nx, ny, 2))))
    ds = diamond_square(2 ** k)[:ny, :nx]
    ds = (ds - ds.min()) * (30.0 / (ds.max() - ds.min()))      # 30 m relief
    x = _centres(nx, dx)[None, :]
    y = _centres(ny, dy)[:, None]
    z = ds + 0.002 * (Lx - x) + 0.01 * np.abs(y - 0.5 * Ly)
    if channel_cells is None:
        channel_cells = 20 if ny >= 80 else max(2, ny // 4)
    j0 = ny // 2 - channel_cells // 2
    j1 = j0 + channel_cells
    z[j0:j1, :] = -3.0 + 0.002 * (Lx - x)[0]
    n_field = 0.02 + 0.06 * rng.uniform(4, nx * ny).reshape(ny, nx)
    width = channel_cells * dy
    qscale = width / 40.0                                       # same unit discharge as the full size
    bc = {"W": "inflow", "E": "free", "S": "wall", "N": "wall"}
    inflow = {"W": Inflow(k0=j0, k1=j1, hydro_t=[0.0, 600.0], hydro_q=[50.0 * qscale, 200.0 * qscale])}
    return SwofConfig(name="cfg3", nx=nx, ny=ny, dx=dx, dy=dy, fric_law="manning", fric_coef=0.05,
                      fric_field=np.ascontiguousarray(n_field), ga=GreenAmpt(), rain_t=[0.0],
                      rain_rate=[mm_per_h(20.0)], bc=bc, inflow=inflow, steps=steps,
                      z=np.ascontiguousarray(z), h=_zeros(ny, nx), hu=_zeros(ny, nx), hv=_zeros(ny, nx),
                      vinf=np.full((ny, nx), GreenAmpt().vinf0))


# ----------------------------------------------------------------------------------------------
# cfg4: 8192^2, dx 1 m, cfg2's sinusoid draws rescaled to 20 m relief, 40% random puddles
#       (mask stream 2, depth stream 3), rain 30 mm/h, GA, Manning 0.04, 4 walls, 1000 steps
# ----------------------------------------------------------------------------------------------
def make_cfg4(nx: int = 8192, ny: int = 8192, steps: int = 1000) -> SwofConfig:
    dx = dy = 1.0
    z = _sinusoid_terrain(nx, ny, dx, dy)
    zmin, zmax = z.min(), z.max()
    z -= zmin
    z *= 20.0 / (zmax - zmin)
    h = np.empty((ny, nx), dtype=np.float64)
    rows = max(1, (1 << 22) // nx)
    for j0 in range(0, ny, rows):
        j1 = min(ny, j0 + rows)
        n0, n = j0 * nx, (j1 - j0) * nx
        mask = rng.uniform(2, n, n0) < 0.4
        depth = 0.3 * rng.uniform(3, n, n0)
        h[j0:j1] = np.where(mask, depth, 0.0).reshape(j1 - j0, nx)
    return SwofConfig(name="cfg4", nx=nx, ny=ny, dx=dx, dy=dy, fric_law="manning", fric_coef=0.04,
                      ga=GreenAmpt(), rain_t=[0.0], rain_rate=[mm_per_h(30.0)], steps=steps,
                      z=z, h=h, hu=_zeros(ny, nx), hv=_zeros(ny, nx), vinf=np.full((ny, nx), GreenAmpt().vinf0))


_MAKERS = {"cfg0": make_cfg0, "cfg1": make_cfg1, "cfg2": make_cfg2, "cfg3": make_cfg3, "cfg4": make_cfg4}


def _cached(name, nx, ny, kw):
    """Optional on-disk cache of generated inputs (env SWOF_WORKLOAD_CACHE=dir; used by tools/ab.sh so that
    repeated bench runs in one GPU session do not regenerate 8192^2 rasters)."""
    import os
    import pickle
    d = os.environ.get("SWOF_WORKLOAD_CACHE")
    if not d:
        return None, None
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, f"{name}_{nx}_{ny}_{sorted(kw.items())}.pkl".replace(" ", ""))
    if os.path.exists(path):
        with open(path, "rb") as f:
            return pickle.load(f), path
    return None, path


def make(name: str, nx: Optional[int] = None, ny: Optional[int] = None, **kw) -> SwofConfig:
    """Build workload `name` at full size, or the same recipe at (nx, ny)."""
    cfg, path = _cached(name, nx, ny, kw)
    if cfg is not None:
        return cfg
    cfg = _make(name, nx, ny, **kw)
    if path is not None:
        import pickle
        with open(path, "wb") as f:
            pickle.dump(cfg, f, protocol=4)
    return cfg


def _make(name: str, nx: Optional[int] = None, ny: Optional[int] = None, **kw) -> SwofConfig:
    fn = _MAKERS[name]
    if nx is not None:
        kw["nx"] = nx
    if ny is not None:
        kw["ny"] = ny
    return fn(**kw)
