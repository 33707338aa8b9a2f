"""Pins of the oracle's FREE (supercritical outflow) boundary ghost (§2.2: "free boundary
conditions are considered for supercritical outflow"; SURVEY.md §8a a1 / DESIGN.md §3 reading: zero-gradient
copy of interior layer 0 -- h, q and z -- into both ghost layers).

What pins it, independently of the oracle's own formulas:
* a zero-gradient ghost makes the boundary face see the boundary cell's own state on both sides (all MUSCL
  slopes there are 0), and HLL is consistent (F(U, U) = F(U)), so the flux through a FREE side is the exact
  physical flux of the boundary cell, (q_n, q_n u_n + g h^2/2, q_n u_t).  Interior faces telescope, so one
  stage changes the totals by exactly -lambda (F_out - F_in) of those closed forms;
* a uniform flow on a flat bed with FREE sides is an exact steady state (every face carries the same flux).

Mutations these catch (checked by hand against swof_oracle.c fill_ghosts): copying interior layer 1 instead
of layer 0, negating the normal discharge (the WALL rule), dropping the copy of z, copying the transverse
discharge with the wrong sign, a WALL instead of FREE.
"""
import numpy as np
import pytest

import oracle
from workloads.configs import SwofConfig

G = 9.81


def _cfg(nx, ny, bc, z, h, hu, hv, dx=1.0, dy=1.0):
    c = SwofConfig(name="freepin", nx=nx, ny=ny, dx=dx, dy=dy, bc=bc)
    c.z, c.h, c.hu, c.hv = z, h, hu, hv
    return c


def _stage(cfg, dt):
    P = oracle.params_from_config(cfg)
    h, hu, hv, _, _ = oracle.stage(P, cfg.z, None, cfg.h, cfg.hu, cfg.hv, None, 0.0, dt)
    return h, hu, hv


def _phys_flux(h, qn, qt):
    """Exact physical flux of a wet cell state along its normal: (q_n, q_n u_n + g h^2 / 2, q_n u_t)."""
    un = qn / h
    return qn, qn * un + 0.5 * G * h * h, qn * (qt / h)


def _ritter_row(nx, dx, t, x0, h0=2.0):
    """Ritter's dry-bed dam-break solution (textbook closed form) at time t on cell centres: wet fan
    h = (2 c0 - (x - x0)/t)^2 / (9 g), u = 2/3 ((x - x0)/t + c0) for -c0 t < x - x0 < 2 c0 t."""
    c0 = np.sqrt(G * h0)
    x = (np.arange(nx) + 0.5) * dx
    xi = (x - x0) / t
    h = np.where(xi <= -c0, h0, np.where(xi >= 2 * c0, 0.0, (2 * c0 - xi) ** 2 / (9 * G)))
    u = np.where(xi <= -c0, 0.0, np.where(xi >= 2 * c0, 0.0, 2.0 / 3.0 * (xi + c0)))
    return h, u


def test_free_uniform_flow_is_steady_bitwise():
    """Uniform (h, hu, hv) = (1, 0.5, 0.2) on a flat bed, FREE on all four sides, frictionless: one full Heun
    step leaves the state unchanged bit for bit.  A wall or a negated ghost discharge on any side breaks it."""
    nx, ny = 12, 9
    z = np.zeros((ny, nx))
    h = np.ones((ny, nx))
    hu = np.full((ny, nx), 0.5)
    hv = np.full((ny, nx), 0.2)
    cfg = _cfg(nx, ny, {s: "free" for s in "WESN"}, z, h, hu, hv)
    r = oracle.run(cfg, nsteps=1)
    assert r["rc"] == 0 and r["steps"] == 1
    for k, ref in (("h", h), ("hu", hu), ("hv", hv)):
        assert np.array_equal(r[k], ref), k
    # control: the same flow against a wall on the east side is not steady
    cw = _cfg(nx, ny, {"W": "free", "E": "wall", "S": "free", "N": "free"}, z, h, hu, hv)
    rw = oracle.run(cw, nsteps=1)
    assert not np.array_equal(rw["h"], h)


@pytest.mark.parametrize("axis", ["x", "y"])
@pytest.mark.parametrize("case", ["ritter_exit_east", "smooth_sloped_both", "ritter_exit_west"])
def test_free_boundary_flux_is_cell_flux(axis, case):
    """One predictor stage of a 1-D problem (periodic in the transverse direction, a single row/column) with
    FREE ends: the totals of h and of the transverse discharge change by exactly -lambda (F_out - F_in),
    F the closed-form physical flux of the two boundary cells; on a flat bed the normal discharge too."""
    n, dx = 64, 1.0
    rng = np.random.default_rng(1307)
    if case.startswith("ritter"):
        # the Ritter fan at t = 6 s with the dam at x0 = 20 m: the front (x0 + 2 c0 t = 73 m) has left the
        # 64 m domain through the east side, supercritical there (u > sqrt(g h))
        h, un = _ritter_row(n, dx, 6.0, 20.0)
        z = np.zeros(n)
        ut = 0.1 + 0.05 * np.sin(np.arange(n) / 5.0)
        if case == "ritter_exit_west":
            h, un, ut = h[::-1].copy(), -un[::-1], ut[::-1].copy()
        assert np.all(h > 0.0)
        flat = True
    else:
        x = np.arange(n) + 0.5
        h = 1.0 + 0.3 * np.sin(x / 7.0) + 0.05 * rng.uniform(size=n)
        un = 0.4 + 0.2 * np.cos(x / 9.0)
        ut = 0.2 * np.sin(x / 4.0)
        z = 0.5 + 0.01 * x          # a sloped bed: a dropped z copy changes the boundary face's depths
        flat = False
    qn, qt = h * un, h * ut
    dt = 0.01
    if axis == "x":
        bc = {"W": "free", "E": "free", "S": "periodic", "N": "periodic"}
        cfg = _cfg(n, 1, bc, z[None, :].copy(), h[None, :].copy(), qn[None, :].copy(), qt[None, :].copy(), dx=dx)
        h1, qn1, qt1 = (a[0] for a in _stage(cfg, dt))
    else:
        bc = {"W": "periodic", "E": "periodic", "S": "free", "N": "free"}
        cfg = _cfg(1, n, bc, z[:, None].copy(), h[:, None].copy(), qt[:, None].copy(), qn[:, None].copy(), dy=dx)
        h1, qt1, qn1 = (a[:, 0] for a in _stage(cfg, dt))
    lam = dt / dx
    Fin = _phys_flux(h[0], qn[0], qt[0])
    Fout = _phys_flux(h[-1], qn[-1], qt[-1])
    scale = np.sum(h)
    dm = np.sum(h1) - np.sum(h)
    assert abs(dm - (-lam * (Fout[0] - Fin[0]))) <= 1e-13 * scale, (dm, -lam * (Fout[0] - Fin[0]))
    dtr = np.sum(qt1) - np.sum(qt)
    assert abs(dtr - (-lam * (Fout[2] - Fin[2]))) <= 1e-13 * scale, (dtr, -lam * (Fout[2] - Fin[2]))
    if flat:    # no bed-slope sources: the normal momentum telescopes as well
        dn = np.sum(qn1) - np.sum(qn)
        assert abs(dn - (-lam * (Fout[1] - Fin[1]))) <= 1e-12 * scale, (dn, -lam * (Fout[1] - Fin[1]))
    # and mass crosses a FREE side materially in every case (a wall would carry none)
    assert max(abs(Fout[0]), abs(Fin[0])) > 1e-1


def test_free_boundary_flux_ignores_second_interior_layer():
    """Only layer 0 feeds a FREE ghost: changing interior cell 1 changes the update of cells 0..3 (the
    stencil) but not the flux through the boundary face, so the total-mass change stays -lambda (F_out - F_in)
    with the boundary cells' own states (a layer-1 copy would move it by O(lambda |q_1 - q_0|))."""
    n = 16
    x = np.arange(n) + 0.5
    h = 1.0 + 0.2 * np.sin(x / 3.0)
    q = 0.5 + 0.3 * np.cos(x / 2.0)
    z = 0.2 + 0.02 * x
    for bump in (0.0, 0.25):
        h2, q2 = h.copy(), q.copy()
        h2[1] += bump
        q2[1] -= bump
        h2[-2] += bump
        q2[-2] += bump
        bc = {"W": "free", "E": "free", "S": "periodic", "N": "periodic"}
        cfg = _cfg(n, 1, bc, z[None, :].copy(), h2[None, :].copy(), q2[None, :].copy(), np.zeros((1, n)))
        h1, _, _ = _stage(cfg, 0.01)
        dm = np.sum(h1) - np.sum(h2)
        assert abs(dm - (-0.01 * (q2[-1] - q2[0]))) <= 1e-13 * np.sum(h2), (bump, dm)
