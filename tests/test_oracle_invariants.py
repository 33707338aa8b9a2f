"""T2/T3: stage pins and whole-scheme invariants of the oracle (SURVEY.md §8c c3 pins N3-N9).

What pins what (a plausible mistake anywhere -- dropped term, wrong sign or index, transposed
operand -- fails at least one of these):
  * N3 3x3 closed form      -> MUSCL limiting, hydrostatic recon, HLL, wall ghosts, update signs, CFL
  * N4 lake at rest         -> well-balancing: S_L/S_R, Fc, eta-based hydrostatic recon, wall z mirror
  * N5 mass                 -> conservative update, wall mass flux = 0, rain, GA, Heun averaging of V
  * N6 positivity           -> hydrostatic recon + CFL; clamps only at round-off level
  * N7 symmetry             -> x/y roles of every index and operand (transpose, reflection)
  * N8 uniform recurrences  -> friction law, Heun combiner, rain/GA recurrence
  * N9 1D reductions        -> consistency + convergence against Ritter/Stoker closed forms
  * inflow mass             -> inflow ghost (critical depth, discharge) against Q(t) dt
"""
import json
import math
import os

from decimal import Decimal, getcontext

import numpy as np
import pytest

import oracle
from workloads import make
from workloads.configs import GreenAmpt, Inflow, SwofConfig

G = 9.81
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def flat_cfg(nx, ny, **kw):
    kw.setdefault("dx", 1.0)
    kw.setdefault("dy", kw["dx"])
    cfg = SwofConfig(name="t", nx=nx, ny=ny, **kw)
    z = np.zeros((ny, nx))
    cfg.z, cfg.h, cfg.hu, cfg.hv = z, z.copy(), z.copy(), z.copy()
    return cfg


# ---------------------------------------------------------------- N3: 3x3 predictor stage
def test_stage_3x3_closed_form():
    ref = gold("stage3x3.json")
    cfg = flat_cfg(3, 3, cfl=0.4)
    cfg.h = np.ones((3, 3))
    cfg.h[1, 1] = 2.0
    P = oracle.params_from_config(cfg)
    # the pin's dt is n_CFL dx / max(|u| + sqrt(g h)) = 0.4/sqrt(2g); under the 2D sum form (Q17)
    # with a_x = a_y the CFL dt is exactly half of it
    dt_cfl, ax, ay = oracle.cfl_dt(P, cfg.h, cfg.hu, cfg.hv)
    assert ax == ay == math.sqrt(2 * G) and dt_cfl == ref["dt"] / 2
    dt = ref["dt"]
    assert abs(dt - 0.4 / math.sqrt(2 * G)) <= 1e-17
    h, hu, hv, _, cnt = oracle.stage(P, cfg.z, None, cfg.h, cfg.hu, cfg.hv, None, 0.0, dt)
    np.testing.assert_allclose(h, np.array(ref["h_after"]), rtol=0, atol=2e-15)
    assert abs(h.sum() - 10.0) <= 1e-14
    w = ref["hu_west_edge_centre"]
    # west / east edge centres carry -+0.6644... in hu; south / north in hv; everything else 0
    assert abs(hu[1, 0] - w) <= 1e-15 and abs(hu[1, 2] + w) <= 1e-15
    assert abs(hv[0, 1] - w) <= 1e-15 and abs(hv[2, 1] + w) <= 1e-15
    mask = np.ones((3, 3), bool)
    mask[1, 0] = mask[1, 2] = False
    assert np.all(hu[mask] == 0)
    mask = np.ones((3, 3), bool)
    mask[0, 1] = mask[2, 1] = False
    assert np.all(hv[mask] == 0)


# ---------------------------------------------------------------- N4: C-property (lake at rest)
def lake_with_islands(nx=64, ny=64, fric="none", coef=0.0):
    cfg = flat_cfg(nx, ny, fric_law=fric, fric_coef=coef)
    x = (np.arange(nx) + 0.5)[None, :]
    y = (np.arange(ny) + 0.5)[:, None]
    z = 0.8 * np.exp(-((x - 40) ** 2 + (y - 24) ** 2) / 60.0) + 0.3 * np.exp(-((x - 16) ** 2 + (y - 44) ** 2) / 20.0)
    z += 0.002 * x                      # a tilted floor too
    C = 0.5
    cfg.z = np.ascontiguousarray(z)
    cfg.h = np.maximum(0.0, C - z)
    return cfg


@pytest.mark.parametrize("fric,coef", [("none", 0.0), ("manning", 0.03)])
def test_lake_at_rest_with_islands(fric, coef):
    cfg = lake_with_islands(fric=fric, coef=coef)
    islands = cfg.h == 0
    assert islands.sum() > 20
    r = oracle.run(cfg, nsteps=1000)
    assert r["rc"] == 0 and r["steps"] == 1000
    assert np.max(np.abs(r["h"] - cfg.h)) <= 1e-12
    assert np.max(np.abs(r["hu"])) <= 1e-12 and np.max(np.abs(r["hv"])) <= 1e-12
    assert np.all(r["h"][islands] == 0.0)          # islands stay exactly dry
    assert r["counters"].clamps == 0


# ---------------------------------------------------------------- N5: mass
def test_mass_walls_cfg0():
    cfg = make("cfg0")
    m0 = oracle.pairwise_sum(cfg.h)
    r = oracle.run(cfg)
    assert r["steps"] == 200
    assert abs(oracle.pairwise_sum(r["h"]) - m0) <= 1e-12 * m0
    assert r["counters"].clamps == 0


def test_mass_budget_rain_green_ampt():
    """Walls + rain + GA: sum(h + V) grows by exactly the Heun-averaged rain, sum_n dt_n (R(t_n) +
    R(t_n + dt_n))/2 per cell, plus half the clamped mass (Q12, Q17); budget to 1e-12 relative."""
    cfg = make("cfg4", nx=48, ny=40, steps=150)
    cfg.rain_t, cfg.rain_rate = [0.0, 5.0], [5e-4, 1e-4]   # a rain change inside the run
    P = oracle.params_from_config(cfg)
    w0 = oracle.pairwise_sum(cfg.h) + oracle.pairwise_sum(cfg.vinf)
    r = oracle.run(cfg)
    t = 0.0
    rain = 0.0
    for dt in r["dt"]:
        rain += dt * (oracle.rain_rate(P, t) + oracle.rain_rate(P, t + dt)) * 0.5
        t += dt
    assert t == r["t"] and t > 5.0
    w1 = oracle.pairwise_sum(r["h"]) + oracle.pairwise_sum(r["v"])
    budget = w0 + rain * cfg.cells + 0.5 * r["counters"].clamped_mass
    assert abs(w1 - budget) <= 1e-12 * w1
    assert r["counters"].ga_capped > 0 and np.all(r["v"] >= cfg.vinf)


# ---------------------------------------------------------------- N6: positivity through wet/dry fronts
@pytest.mark.parametrize("name,nx,ny,steps", [("cfg1", 128, 48, 300), ("cfg4", 64, 64, 200), ("cfg2", 96, 64, 300)])
def test_positivity(name, nx, ny, steps):
    cfg = make(name, nx=nx, ny=ny)
    cfg.steps, cfg.t_end = steps, None
    r = oracle.run(cfg)
    assert r["rc"] == 0 and r["steps"] == steps
    assert np.all(r["h"] >= 0.0) and np.all(np.isfinite(r["hu"])) and np.all(np.isfinite(r["hv"]))
    vol = oracle.pairwise_sum(r["h"]) + (oracle.pairwise_sum(r["v"]) if r["v"] is not None else 0)
    assert r["counters"].clamped_mass <= 1e-15 * max(vol, 1.0)


# ---------------------------------------------------------------- N7: symmetry
def test_transpose_symmetry_bitwise():
    cfg = make("cfg0", steps=60)
    r = oracle.run(cfg)
    assert np.array_equal(r["h"], r["h"].T)
    assert np.array_equal(r["hu"], r["hv"].T)


def test_reflection_symmetry():
    """Centred hump on a flat walled box: x -> -x reflection maps h(i) to h(n-1-i), hu to -hu."""
    cfg = flat_cfg(40, 24, fric_law="manning", fric_coef=0.03)
    x = (np.arange(40) + 0.5)[None, :]
    y = (np.arange(24) + 0.5)[:, None]
    cfg.h = 1.0 + 0.3 * np.exp(-((x - 20.0) ** 2 + (y - 9.0) ** 2) / 8.0)
    r = oracle.run(cfg, nsteps=80)
    assert np.array_equal(r["h"], r["h"][:, ::-1])
    assert np.array_equal(r["hu"], -r["hu"][:, ::-1])
    assert np.array_equal(r["hv"], r["hv"][:, ::-1])


# ---------------------------------------------------------------- N8: uniform-state recurrences
def uniform_periodic(law, coef, h=1.0, q=1.0):
    cfg = flat_cfg(8, 6, fric_law=law, fric_coef=coef,
                   bc={"W": "periodic", "E": "periodic", "S": "periodic", "N": "periodic"})
    cfg.h = np.full((6, 8), h)
    cfg.hu = np.full((6, 8), q)
    return cfg


def test_uniform_friction_recurrence():
    ref = gold("uniform_recurrences.json")
    for law, key, coef in (("manning", "manning", "n"), ("darcy_weisbach", "darcy", "f")):
        ex = ref[key]
        cfg = uniform_periodic(law, ex[coef], ex["h"], ex["q"])
        r = oracle.run(cfg, nsteps=1, dt_forced=ex["dt"])
        assert np.all(r["hu"] == r["hu"][0, 0]) and np.all(r["h"] == 1.0) and np.all(r["hv"] == 0)
        assert abs(r["hu"][0, 0] - ex["q_new"]) <= ex["tol"]
        # scalar recurrence (h = 1 so h^a = 1): q* = q/(1 + dt gCf q), q** = q*/(1 + dt gCf q*)
        gcf = G * ex[coef] ** 2 if law == "manning" else ex[coef] / 8
        q1 = 1.0 / (1.0 + ex["dt"] * gcf * 1.0)
        q2 = q1 / (1.0 + ex["dt"] * gcf * q1)
        assert abs(r["hu"][0, 0] - 0.5 * (1.0 + q2)) <= 2e-16
        if "q_star" in ex:
            assert abs(q1 - ex["q_star"]) < 1e-10 and abs(q2 - ex["q_2star"]) < 1e-10
        # the same closed form in 40-digit decimal arithmetic (h = 1, so h^(4/3) = 1 exactly): the oracle's
        # fp64 result within 1e-14
        getcontext().prec = 40
        D = Decimal
        dgcf = D(repr(G)) * D(repr(ex[coef])) ** 2 if law == "manning" else D(repr(ex[coef])) / 8
        ddt = D(repr(ex["dt"]))
        d1 = D(1) / (D(1) + ddt * dgcf * D(1))
        d2 = d1 / (D(1) + ddt * dgcf * d1)
        want = (D(1) + d2) / 2
        assert abs(D(r["hu"][0, 0]) - want) <= D("1e-14"), (law, r["hu"][0, 0], want)


def test_uniform_rain_green_ampt_recurrence():
    """At rest on a flat periodic bed with rain + GA, each cell follows the pointwise recurrence of
    steps 7-8 of the stage inside Heun."""
    cfg = uniform_periodic("manning", 0.05, h=0.002, q=0.0)
    cfg.ga = GreenAmpt(Ks=2e-6, hf=0.1, A=1.0, dtheta=0.3, vinf0=0.003)
    cfg.vinf = np.full((6, 8), 0.003)
    cfg.rain_t, cfg.rain_rate = [0.0], [3e-5]
    dt = 0.5
    r = oracle.run(cfg, nsteps=3, dt_forced=dt)
    h, V, t = 0.002, 0.003, 0.0
    for _ in range(3):
        def stage(h, V):
            hr = h + 3e-5 * dt
            cap = max(2e-6 * (1.0 + ((0.1 - hr) * 0.3) / V), 0.0) * dt
            inf = min(hr, cap)
            return hr - inf, V + inf
        h1, V1 = stage(h, V)
        h2, V2 = stage(h1, V1)
        h, V = 0.5 * (h + h2), 0.5 * (V + V2)
        t += dt
    assert np.all(r["h"] == h) and np.all(r["v"] == V)
    assert np.all(r["hu"] == 0) and np.all(r["hv"] == 0)


def test_heun_scalar_closed_form():
    """Heun on a linear decay: with DW friction and a tiny dt the uniform recurrence
    approaches q (1 - k dt + (k dt)^2/2) for k = gCf |u|/h, the RK2 closed form."""
    cfg = uniform_periodic("darcy_weisbach", 8.0, h=1.0, q=1e-6)   # |u| tiny: nearly linear decay, k = 1e-6
    r = oracle.run(cfg, nsteps=1, dt_forced=0.1)
    assert np.all(r["h"] == 1.0)
    # semi-implicit stages of a linear ODE q' = -k q, k = (f/8) |u| / h = 1 * 1e-6
    k = 1e-6
    want = 1e-6 * (1 - k * 0.1 + (k * 0.1) ** 2 / 2)
    assert abs(r["hu"][0, 0] - want) <= 1e-6 * 1e-12


# ---------------------------------------------------------------- N9: 1D reductions
def test_y_invariant_data_matches_single_row():
    cfg1 = make("cfg1", nx=96, ny=1, steps=100)
    cfg4 = make("cfg1", nx=96, ny=5, steps=100)
    r1 = oracle.run(cfg1)
    r4 = oracle.run(cfg4)
    for j in range(5):
        assert np.array_equal(r4["h"][j], r1["h"][0])
        assert np.array_equal(r4["hu"][j], r1["hu"][0])
    assert np.all(r4["hv"] == 0)
    assert np.array_equal(r4["dt"], r1["dt"])


def ritter(x, t, h0, x0):
    c0 = math.sqrt(G * h0)
    xi = (x - x0) / t
    h = np.where(xi <= -c0, h0, np.where(xi >= 2 * c0, 0.0, (2 * c0 - xi) ** 2 / (9 * G)))
    return h


def stoker(x, t, h0, hr, x0):
    c0, cr = math.sqrt(G * h0), math.sqrt(G * hr)
    # middle state: u_m from the rarefaction = u_m from the shock (Rankine-Hugoniot), solved by bisection
    def f(hm):
        return 2 * (c0 - math.sqrt(G * hm)) - (hm - hr) * math.sqrt(0.5 * G * (hm + hr) / (hm * hr))
    lo, hi = hr, h0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if f(mid) > 0:
            lo = mid
        else:
            hi = mid
    hm = 0.5 * (lo + hi)
    um = 2 * (c0 - math.sqrt(G * hm))
    s = hm * um / (hm - hr)
    cm = math.sqrt(G * hm)
    xi = (x - x0) / t
    h = np.where(xi <= -c0, h0, (2 * c0 - xi) ** 2 / (9 * G))
    h = np.where(xi >= um - cm, hm, h)
    h = np.where(xi >= s, hr, h)
    return h


@pytest.mark.parametrize("kind", ["ritter", "stoker"])
def test_dam_break_convergence(kind):
    L, x0, h0, hr, tf = 10.0, 5.0, 1.0, (0.0 if kind == "ritter" else 0.2), 0.5
    errs = []
    for n in (100, 200, 400):
        dx = L / n
        cfg = flat_cfg(n, 1, dx=dx, dy=dx)
        x = (np.arange(n) + 0.5) * dx
        cfg.h = np.where(x < x0, h0, hr)[None, :].copy()
        r = oracle.run(cfg, nsteps=100000, t_end=tf)
        assert r["rc"] == 0 and r["t"] == tf
        exact = ritter(x, tf, h0, x0) if kind == "ritter" else stoker(x, tf, h0, hr, x0)
        errs.append(np.sum(np.abs(r["h"][0] - exact)) * dx)
    assert errs[0] < 0.06                   # L1 error of h over a 10 m reach
    assert errs[1] < errs[0] and errs[2] < errs[1]
    assert errs[0] / errs[2] > 3.0          # ~first order in L1 (kinks and the shock limit it)


# ---------------------------------------------------------------- inflow ghost (Q18)
def test_inflow_mass_rate():
    """Dry flat bed, constant Q on a west segment: one predictor stage adds Q dt of water (the critical
    inflow ghost carries q = Q/W into the domain at Froude number 1)."""
    cfg = flat_cfg(12, 10, bc={"W": "inflow", "E": "wall", "S": "wall", "N": "wall"},
                   inflow={"W": Inflow(k0=3, k1=7, hydro_t=[0.0], hydro_q=[2.0])})
    P = oracle.params_from_config(cfg)
    dt = 0.01
    h, hu, hv, _, _ = oracle.stage(P, cfg.z, None, cfg.h, cfg.hu, cfg.hv, None, 0.0, dt)
    vol = h.sum() * cfg.dx * cfg.dy
    assert abs(vol - 2.0 * dt) <= 1e-13
    assert np.all(h[3:7, 0] > 0) and np.all(h[:3, :] == 0) and np.all(h[7:, :] == 0)
    # ramped hydrograph is evaluated at the stage time
    cfg.inflow["W"] = Inflow(k0=3, k1=7, hydro_t=[0.0, 10.0], hydro_q=[0.0, 4.0])
    P = oracle.params_from_config(cfg)
    h, _, _, _, _ = oracle.stage(P, cfg.z, None, cfg.h, cfg.hu, cfg.hv, None, 5.0, dt)
    assert abs(h.sum() - 2.0 * dt) <= 1e-13


def test_inflow_critical_depth_momentum():
    """Pins the inflow ghost's critical depth h_c = (q^2/g)^(1/3) (Q18) by its momentum flux: on a dry flat
    bed the ghost state (h_c, q) is critical (u = sqrt(g h_c)), so the face takes F(U_L) and one stage adds
    hu = (dt/dx) (q^2/h_c + g h_c^2 / 2) = (dt/dx) 1.5 g h_c^2 to the first cell of every segment row
    (no slopes, no interface source, zero stage-input velocity -> friction factor 1)."""
    cfg = flat_cfg(12, 10, bc={"W": "inflow", "E": "wall", "S": "wall", "N": "wall"}, fric_law="manning",
                   fric_coef=0.03, inflow={"W": Inflow(k0=3, k1=7, hydro_t=[0.0], hydro_q=[2.0])})
    P = oracle.params_from_config(cfg)
    dt = 0.01
    h, hu, hv, _, _ = oracle.stage(P, cfg.z, None, cfg.h, cfg.hu, cfg.hv, None, 0.0, dt)
    q = 2.0 / 4.0                                        # Q / W, W = 4 cells x dy = 1 m
    hc = (q * q / G) ** (1.0 / 3.0)
    want = (dt / cfg.dx) * 1.5 * G * hc * hc
    for j in range(3, 7):
        assert abs(hu[j, 0] - want) <= 1e-13 * want, (hu[j, 0], want)
        assert abs(h[j, 0] - (dt / cfg.dx) * q) <= 1e-16
    assert np.all(hu[:, 1:] == 0) and np.all(hv == 0)
