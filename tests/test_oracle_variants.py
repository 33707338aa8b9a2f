"""Pins of the oracle's scheme variants: Rusanov flux, the first-order
scheme with explicit Euler, the CFL on reconstructed values and the Darcy-consistent
Green-Ampt sign (Q15).

Expected values come from tests/golden/variant_pins.json (hand-derived closed forms, cited), from
identities that hold for any correct implementation (consistency, wall symmetry, HLL == Rusanov for
symmetric wave speeds, order-1 faces == cell values), or from the whole-scheme invariants of
test_oracle_invariants.py (C-property, mass, positivity, symmetry, dam-break convergence against
Ritter/Stoker) re-run under each variant.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from workloads import make
from workloads.configs import GreenAmpt

from test_oracle_invariants import flat_cfg, lake_with_islands, ritter, stoker

G = 9.81
with open(os.path.join(os.path.dirname(__file__), "golden", "variant_pins.json")) as f:
    VAR = json.load(f)


def face_in(h, un, ut, z=0.0):
    return [h, h + z, z, un, ut]


# ---------------------------------------------------------------- Rusanov face
def test_rusanov_worked_example():
    ex = VAR["rusanov_subcritical"]
    d = oracle.face_rusanov(face_in(*ex["L"]), face_in(*ex["R"]))
    assert d["branch"] == 3
    assert abs(d["c"] - ex["c"]) <= 1e-15 * ex["c"]
    for k, want in zip(("Fm", "Fn", "Ft"), ex["F"]):
        assert abs(d[k] - want) <= 2e-15 * abs(want), (k, d[k], want)
    # interface sources are the flux-independent hydrostatic terms (flat bed: 0)
    assert d["SL"] == 0.0 and d["SR"] == 0.0


@pytest.mark.parametrize("h,un,ut", [(1.0, 0.3, -0.2), (0.2, -4.0, 1.0), (2.5, 0.0, 0.0), (1e-3, 7.0, 3.0)])
def test_rusanov_consistency(h, un, ut):
    """F(U, U) = F(U): the dissipation term vanishes exactly."""
    d = oracle.face_rusanov(face_in(h, un, ut), face_in(h, un, ut))
    q = h * un
    assert d["Fm"] == q
    assert d["Fn"] == q * un + 0.5 * G * (h * h)
    assert d["Ft"] == q * ut


def test_rusanov_wall_and_dry():
    # mirror states (normal velocity negated): zero mass flux exactly
    for h, un, ut in ((1.0, 0.7, 0.1), (0.3, -2.0, 0.5)):
        d = oracle.face_rusanov(face_in(h, un, ut), face_in(h, -un, ut))
        assert d["Fm"] == 0.0
    d = oracle.face_rusanov(face_in(0.0, 0.0, 0.0), face_in(1e-13, 0.0, 0.0))
    assert d["branch"] == 0 and d["Fm"] == d["Fn"] == d["Ft"] == 0.0


@pytest.mark.parametrize("hl,hr", [(1.0, 0.5), (0.2, 2.0), (1.0, 0.0)])
def test_rusanov_equals_hll_for_symmetric_speeds(hl, hr):
    """With both states at rest HLL's speeds are c1 = -c2 = -max(c_L, c_R), and the HLL formula
     reduces algebraically to the Rusanov form with c = c2: they agree to rounding."""
    a = oracle.face(face_in(hl, 0.0, 0.0), face_in(hr, 0.0, 0.0))
    b = oracle.face_rusanov(face_in(hl, 0.0, 0.0), face_in(hr, 0.0, 0.0))
    assert a["branch"] == 3 and a["c1"] == -a["c2"] and b["c"] == a["c2"]
    for k in ("Fm", "Fn", "Ft"):
        assert abs(a[k] - b[k]) <= 4e-16 * max(1.0, abs(a[k])), k


def variant(cfg, **kw):
    for k, v in kw.items():
        setattr(cfg, k, v)
    return cfg


VARIANTS = [dict(flux="rusanov"), dict(order=1, cfl=1.0), dict(cfl_mode="face"),
            dict(flux="rusanov", order=1, cfl=1.0, cfl_mode="face")]


# ---------------------------------------------------------------- whole-scheme invariants per variant
@pytest.mark.parametrize("kw", VARIANTS)
def test_variant_lake_at_rest(kw):
    cfg = variant(lake_with_islands(fric="manning", coef=0.03), **kw)
    islands = cfg.h == 0
    r = oracle.run(cfg, nsteps=300)
    assert r["rc"] == 0 and r["steps"] == 300
    assert np.max(np.abs(r["h"] - cfg.h)) <= 1e-12
    assert np.max(np.abs(r["hu"])) <= 1e-12 and np.max(np.abs(r["hv"])) <= 1e-12
    assert np.all(r["h"][islands] == 0.0) and r["counters"].clamps == 0


@pytest.mark.parametrize("kw", VARIANTS)
def test_variant_mass_and_symmetry(kw):
    cfg = variant(make("cfg0", steps=60), **kw)
    m0 = oracle.pairwise_sum(cfg.h)
    r = oracle.run(cfg)
    assert r["steps"] == 60
    assert abs(oracle.pairwise_sum(r["h"]) - m0) <= 1e-12 * m0
    assert np.array_equal(r["h"], r["h"].T) and np.array_equal(r["hu"], r["hv"].T)


@pytest.mark.parametrize("kw", VARIANTS)
def test_variant_positivity_wet_dry(kw):
    cfg = variant(make("cfg4", nx=48, ny=40, steps=120), **kw)
    r = oracle.run(cfg)
    assert r["rc"] == 0 and r["steps"] == 120
    assert np.all(r["h"] >= 0.0) and np.all(np.isfinite(r["hu"]))
    vol = oracle.pairwise_sum(r["h"]) + oracle.pairwise_sum(r["v"])
    assert r["counters"].clamped_mass <= 1e-15 * vol


@pytest.mark.parametrize("kw,kind,err100,ratio", [(dict(flux="rusanov"), "ritter", 0.07, 3.5),
                                                  (dict(flux="rusanov"), "stoker", 0.07, 3.5),
                                                  (dict(order=1, cfl=1.0), "ritter", 0.11, 2.2),
                                                  (dict(order=1, cfl=1.0), "stoker", 0.12, 2.2)])
def test_variant_dam_break_convergence(kw, kind, err100, ratio):
    """L1(h) against Ritter (dry) / Stoker (wet) at N = 100, 200, 400: second order (Rusanov) converges
    at ~first order in L1 (the kinks and the shock limit it), the first-order scheme at ~0.7."""
    L, x0, h0, hr, tf = 10.0, 5.0, 1.0, (0.0 if kind == "ritter" else 0.2), 0.5
    errs = []
    for n in (100, 200, 400):
        dx = L / n
        cfg = variant(flat_cfg(n, 1, dx=dx, dy=dx), **kw)
        x = (np.arange(n) + 0.5) * dx
        cfg.h = np.where(x < x0, h0, hr)[None, :].copy()
        r = oracle.run(cfg, nsteps=100000, t_end=tf)
        assert r["rc"] == 0 and r["t"] == tf
        exact = ritter(x, tf, h0, x0) if kind == "ritter" else stoker(x, tf, h0, hr, x0)
        errs.append(np.sum(np.abs(r["h"][0] - exact)) * dx)
    assert errs[0] < err100
    assert errs[1] < errs[0] and errs[2] < errs[1]
    assert errs[0] / errs[2] > ratio


# ---------------------------------------------------------------- first order + Euler
def test_first_order_3x3_closed_form():
    """The N3 pin's limiter zeroes every slope, so its closed form is also the first-order stage."""
    with open(os.path.join(os.path.dirname(__file__), "golden", "stage3x3.json")) as f:
        ref = json.load(f)
    cfg = variant(flat_cfg(3, 3, cfl=1.0), order=1)
    cfg.h = np.ones((3, 3))
    cfg.h[1, 1] = 2.0
    P = oracle.params_from_config(cfg)
    h, hu, hv, _, _ = oracle.stage(P, cfg.z, None, cfg.h, cfg.hu, cfg.hv, None, 0.0, ref["dt"])
    np.testing.assert_allclose(h, np.array(ref["h_after"]), rtol=0, atol=2e-15)
    assert abs(hu[1, 0] - ref["hu_west_edge_centre"]) <= 1e-15


def test_first_order_step_is_one_stage():
    """Explicit Euler: one order-1 step equals one stage S(U^n; t^n, dt) with the step's CFL dt."""
    cfg = variant(make("cfg4", nx=40, ny=32, steps=1), order=1, cfl=1.0)
    P = oracle.params_from_config(cfg)
    dt, _, _ = oracle.cfl_dt(P, cfg.h, cfg.hu, cfg.hv)
    h, hu, hv, v, _ = oracle.stage(P, cfg.z, None, cfg.h, cfg.hu, cfg.hv, cfg.vinf, 0.0, dt)
    r = oracle.run(cfg)
    assert r["dt"][0] == dt
    for a, b in ((r["h"], h), (r["hu"], hu), (r["hv"], hv), (r["v"], v)):
        assert np.array_equal(a, b)


def test_first_order_faces_are_cell_values():
    cfg = variant(make("cfg2", nx=24, ny=20), order=1)
    cfg.h = np.abs(np.sin(np.arange(cfg.cells).reshape(cfg.ny, cfg.nx))) + 0.1
    P = oracle.params_from_config(cfg)
    _, ax1, ay1 = oracle.cfl_dt_face(P, cfg.z, cfg.h, cfg.hu, cfg.hv)
    _, ax0, ay0 = oracle.cfl_dt(P, cfg.h, cfg.hu, cfg.hv)
    assert ax1 == ax0 and ay1 == ay0      # order 1: reconstructed values are the cell values


# ---------------------------------------------------------------- CFL on reconstructed values
def test_face_cfl_worked_example():
    ex = VAR["cfl_face_1d"]
    cfg = variant(flat_cfg(3, 1), cfl_mode="face")
    cfg.h = np.array([ex["h"]])
    cfg.hu = np.array([ex["h"]]) * np.array([ex["u"]])
    P = oracle.params_from_config(cfg)
    _, ax, ay = oracle.cfl_dt_face(P, cfg.z, cfg.h, cfg.hu, cfg.hv)
    _, axc, _ = oracle.cfl_dt(P, cfg.h, cfg.hu, cfg.hv)
    assert abs(ax - ex["a_face"]) <= 2e-15 * ex["a_face"]
    assert abs(axc - ex["a_cell"]) <= 2e-15 * ex["a_cell"]
    assert ax > axc
    assert abs(ay - math.sqrt(3 * G)) <= 1e-15 * ay     # y: one row, mirrored ghosts -> zero slopes


def test_face_cfl_at_rest_bounded_by_cell_cfl():
    """At rest the minmod faces stay within the neighbours' range, so a_face <= a_cell."""
    cfg = make("cfg0")
    P = oracle.params_from_config(variant(cfg, cfl_mode="face"))
    _, ax, ay = oracle.cfl_dt_face(P, cfg.z, cfg.h, cfg.hu, cfg.hv)
    _, axc, ayc = oracle.cfl_dt(P, cfg.h, cfg.hu, cfg.hv)
    assert 0 < ax <= axc and 0 < ay <= ayc


# ---------------------------------------------------------------- Green-Ampt forms (Q15)
def test_green_ampt_forms_worked_example():
    ex = VAR["green_ampt_forms"]
    cfg = flat_cfg(2, 2)
    cfg.ga = GreenAmpt(Ks=ex["Ks"], hf=ex["hf"], A=ex["A"], dtheta=ex["dtheta"], vinf0=ex["V"])
    for form, cap in (("printed", ex["cap_printed"]), ("darcy", ex["cap_darcy"])):
        cfg.ga_form = form
        P = oracle.params_from_config(cfg)
        h_out, V_out = oracle.green_ampt(P, ex["h_over"], ex["V"], ex["dt"])
        assert abs((V_out - ex["V"]) - cap) <= 1e-18                # capacity-limited (V_out - V: ulp(V) ~ 4e-19)
        assert abs(h_out - (ex["h_over"] - cap)) <= 1e-16
        # ponded depth below the capacity: everything infiltrates in both forms
        h_out, V_out = oracle.green_ampt(P, 1e-7, ex["V"], ex["dt"])
        assert h_out == 0.0 and V_out == ex["V"] + 1e-7


def test_green_ampt_darcy_mass_budget():
    cfg = variant(make("cfg4", nx=40, ny=32, steps=100), ga_form="darcy")
    P = oracle.params_from_config(cfg)
    w0 = oracle.pairwise_sum(cfg.h) + oracle.pairwise_sum(cfg.vinf)
    r = oracle.run(cfg)
    t, rain = 0.0, 0.0
    for dt in r["dt"]:
        rain += dt * (oracle.rain_rate(P, t) + oracle.rain_rate(P, t + dt)) * 0.5
        t += dt
    w1 = oracle.pairwise_sum(r["h"]) + oracle.pairwise_sum(r["v"])
    assert abs(w1 - (w0 + rain * cfg.cells + 0.5 * r["counters"].clamped_mass)) <= 1e-12 * w1
    # the Darcy form infiltrates at least as much as the printed one (h_over >= 0)
    r0 = oracle.run(variant(make("cfg4", nx=40, ny=32, steps=100), ga_form="printed"))
    assert oracle.pairwise_sum(r["v"]) >= oracle.pairwise_sum(r0["v"])
