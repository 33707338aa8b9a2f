"""Shared helpers for the parity tests (tests only: may use both the oracle and the product)."""
from __future__ import annotations

import copy

import numpy as np

import oracle


def gpu_solver(cfg, graph_steps=0, **kw):
    from paper_1307_4839_b200 import Solver, params_from_config
    s = Solver(params_from_config(cfg, graph_steps=graph_steps), cfg.z, cfg.fric_field, **kw)
    s.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf if cfg.ga is not None else None, 0.0)
    return s


def gpu_run(cfg, nsteps=None, t_end=None, graph_steps=0):
    s = gpu_solver(cfg, graph_steps=graph_steps)
    if t_end is not None:
        s.run(t_end, nsteps if nsteps is not None else 1 << 40)
    else:
        s.step(nsteps)
    out = s.get_state()
    out["dt"] = s.dt_history()
    out["diag"] = s.diag()
    s.close()
    return out


def max_abs(a, b):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) if np.size(a) else 0.0


def compare(g, r, tol, keys=("h", "hu", "hv")):
    """Element-by-element comparison; returns dict of max |diff| and whether all are bitwise equal."""
    res = {k: max_abs(g[k], r[k]) for k in keys}
    res["bitwise"] = all(np.array_equal(g[k], r[k]) for k in keys)
    for k in keys:
        assert res[k] <= tol, (k, res[k], tol)
    return res


def patch_config(cfg, i0, i1, j0, j1):
    """Sub-rectangle [i0,i1) x [j0,j1) of a workload as its own problem: sides on the physical boundary
    keep their boundary condition, cut sides become FREE (their ghosts only reach cells within 4 of the
    cut, which the caller does not compare).  Inflow segments are shifted and, if cut, rescaled so the
    unit discharge Q/W is unchanged."""
    p = copy.copy(cfg)
    p.nx, p.ny = i1 - i0, j1 - j0
    p.bc = dict(cfg.bc)
    p.inflow = {}
    touch = {"W": i0 == 0, "E": i1 == cfg.nx, "S": j0 == 0, "N": j1 == cfg.ny}
    for side in ("W", "E", "S", "N"):
        if not touch[side]:
            p.bc[side] = "free"
    if (cfg.bc["W"] == "periodic" or cfg.bc["S"] == "periodic") and not all(touch.values()):
        raise ValueError("periodic patches need the full extent")
    for side, fl in cfg.inflow.items():
        if not touch[side]:
            continue
        off = j0 if side in ("W", "E") else i0
        n = p.ny if side in ("W", "E") else p.nx
        k0, k1 = max(fl.k0 - off, 0), min(fl.k1 - off, n)
        if k0 >= k1:
            p.bc[side] = "wall"
            continue
        scale = (k1 - k0) / (fl.k1 - fl.k0)
        p.inflow[side] = type(fl)(k0=k0, k1=k1, hydro_t=list(fl.hydro_t), hydro_q=[q * scale for q in fl.hydro_q])
    return p


def oracle_patch_step(cfg, st, t, dt, i, j, R=6):
    """Oracle Heun step with the given dt on the (2R+1)^2 patch of state `st` around cell (i, j).
    Returns (patch slices, outputs, validity mask of cells unaffected by cut sides)."""
    i0, i1 = max(i - R, 0), min(i + R + 1, cfg.nx)
    j0, j1 = max(j - R, 0), min(j + R + 1, cfg.ny)
    p = patch_config(cfg, i0, i1, j0, j1)
    sl = (slice(j0, j1), slice(i0, i1))
    P = oracle.params_from_config(p)
    fric = cfg.fric_field[sl] if cfg.fric_field is not None else None
    v = st["v"][sl] if cfg.ga is not None else None
    r = oracle.run(P, z=cfg.z[sl], fric=fric, h=st["h"][sl], hu=st["hu"][sl], hv=st["hv"][sl], v=v, t0=t,
                   nsteps=1, dt_forced=dt)
    assert r["rc"] == 0 and r["steps"] == 1
    valid = np.ones((j1 - j0, i1 - i0), bool)
    if i0 > 0:
        valid[:, :4] = False
    if i1 < cfg.nx:
        valid[:, -4:] = False
    if j0 > 0:
        valid[:4, :] = False
    if j1 < cfg.ny:
        valid[-4:, :] = False
    return sl, r, valid
