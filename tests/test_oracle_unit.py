"""T1: pointwise pins of the oracle against values the paper / SPEC worked examples / closed forms fix.

Every expected value here comes from tests/golden/*.json (cited) or from a closed form evaluated
independently of the oracle (plain Python math on the special case) -- never from the oracle itself.
"""
import json
import math
import os
from decimal import Decimal, getcontext

import numpy as np
import pytest

import oracle

G = 9.81
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


SPEC = gold("spec_examples.json")
FACE = gold("face_pins.json")


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# ---------------------------------------------------------------- minmod / MUSCL
def test_minmod_table():
    for a, b, want in SPEC["minmod"]["cases"]:
        assert oracle.minmod(a, b) == want
    # symmetric, odd, bounded (definition)
    rng = np.random.default_rng(1)
    for a, b in rng.normal(size=(200, 2)):
        m = oracle.minmod(a, b)
        assert m == oracle.minmod(b, a)
        assert oracle.minmod(-a, -b) == -m
        assert abs(m) <= min(abs(a), abs(b))
        assert (m == 0) == (a * b <= 0)


def test_muscl_slopes_and_faces():
    for s3, want in SPEC["muscl_slope"]["cases"]:
        r = oracle.muscl_cell(s3, s3, [0, 0, 0], [0, 0, 0], 0.0)
        # delta = (hp - hm)/2 = 0.5 * minmod(...) with dx = 1, so Ds = hp - hm
        assert r["hp"] - r["hm"] == want
    ex = SPEC["reconstruct_scalar"]
    s = ex["s"]
    r = oracle.muscl_cell([s - ex["Ds"], s, s + ex["Ds"]], [0, 0, 0], [0, 0, 0], [0, 0, 0], 0.0)
    assert [r["hm"], r["hp"]] == ex["faces"]


def test_muscl_monotone_and_mean():
    """Faces lie within the 3-cell range and average to the cell value."""
    rng = np.random.default_rng(2)
    for _ in range(500):
        h3 = rng.uniform(0.1, 2.0, 3)
        r = oracle.muscl_cell(h3, h3, [0, 0, 0], [0, 0, 0], 1.0 / h3[1])
        lo, hi = h3.min(), h3.max()
        for k in ("hm", "hp"):
            assert lo - 1e-15 <= r[k] <= hi + 1e-15
        assert abs(0.5 * (r["hm"] + r["hp"]) - h3[1]) <= 4e-16 * h3[1]


def test_velocity_modification_conserves_discharge():
    """(h_- u_- + h_+ u_+)/2 = h u on wet cells (exact identity, round-off only)."""
    rng = np.random.default_rng(3)
    for _ in range(500):
        h3 = rng.uniform(0.05, 3.0, 3)
        u3 = rng.normal(size=3)
        v3 = rng.normal(size=3)
        z3 = rng.uniform(-1, 1, 3)
        r = oracle.muscl_cell(h3, h3 + z3, u3, v3, 1.0 / h3[1])
        assert abs(0.5 * (r["hm"] * r["um"] + r["hp"] * r["up"]) - h3[1] * u3[1]) <= 1e-14 * (1 + abs(h3[1] * u3[1]))
        assert abs(0.5 * (r["hm"] * r["vm"] + r["hp"] * r["vp"]) - h3[1] * v3[1]) <= 1e-14 * (1 + abs(h3[1] * v3[1]))
        assert abs(0.5 * (r["hm"] + r["hp"]) - h3[1]) <= 1e-15 * h3[1]
        # z deduced from eta - h: z faces average to z on a linear-eta cell pair
        assert r["zm"] == r["em"] - r["hm"] and r["zp"] == r["ep"] - r["hp"]


def test_dry_cell_velocity_unreconstructed():
    r = oracle.muscl_cell([1, 0, 1], [2, 1, 2], [1, 5, 1], [0, 3, 0], 0.0)
    assert r["um"] == r["up"] == 5 and r["vm"] == r["vp"] == 3


# ---------------------------------------------------------------- flux
def test_wave_speeds():
    for h, u, l1, l2 in SPEC["wave_speeds"]["cases"]:
        f = oracle.face([h, h, 0, u, 0], [h, h, 0, u, 0])
        assert rel(f["c1"], l1) < 1e-15 and rel(f["c2"], l2) < 1e-15


def test_physical_flux_consistency():
    """HLL(U, U) = F(U); F = (hu, hu^2 + g h^2/2)."""
    for h, u, fm, fn in SPEC["physical_flux"]["cases"]:
        f = oracle.face([h, h, 0, u, 0], [h, h, 0, u, 0])
        assert rel(f["Fm"], fm) < 1e-15 if fm else f["Fm"] == 0
        assert rel(f["Fn"], fn) < 1e-15


def test_hydrostatic_and_interface_source():
    ex = SPEC["hydrostatic"]
    l = [ex["h_minus"], ex["h_minus"] + ex["z_minus"], ex["z_minus"], 0, 0]
    r = [ex["h_plus"], ex["h_plus"] + ex["z_plus"], ex["z_plus"], 0, 0]
    f = oracle.face(l, r)
    assert f["HL"] == ex["h_L"] and f["HR"] == ex["h_R"]
    s = SPEC["interface_source"]
    assert rel(f["SL"], s["s_left"]) < 1e-15
    assert f["SR"] == 0.0


def test_centered_source():
    ex = SPEC["centered_source"]
    fc = oracle.centered_source(ex["h_faces"][0], ex["h_faces"][1], ex["z_faces"][0], ex["z_faces"][1])
    assert rel(fc, ex["Fc"]) < 1e-15


@pytest.mark.parametrize("case", ["subcritical", "supercritical", "wet_dry"])
def test_hll_face_pins(case):
    c = FACE[case]
    (hl, ul, tl), (hr, ur, tr) = c["L"], c["R"]
    f = oracle.face([hl, hl, 0, ul, tl], [hr, hr, 0, ur, tr])
    for k, want in zip(("Fm", "Fn", "Ft"), c["F"]):
        assert abs(f[k] - want) <= 1e-14 * max(1.0, abs(want)), (k, f[k], want)
    if "c1" in c:
        assert rel(f["c1"], c["c1"]) < 1e-15 and rel(f["c2"], c["c2"]) < 1e-15


def test_hll_closed_forms():
    # subcritical pin closed forms: c1 = -sqrt(g/2), c2 = 1 + sqrt(g)
    f = oracle.face([1, 1, 0, 1, 0.5], [0.5, 0.5, 0, 0, 0])
    assert rel(f["c1"], -math.sqrt(G * 0.5)) < 1e-15 and rel(f["c2"], 1 + math.sqrt(G)) < 1e-15
    # wet/dry: Fm = sqrt(g)/2 (Ritter fan at the face), Fn = g/4
    f = oracle.face([1, 1, 0, 0, 0], [0, 0, 0, 0, 0])
    assert rel(f["Fm"], math.sqrt(G) / 2) < 1e-15 and rel(f["Fn"], G / 4) < 1e-15
    # dry/dry -> zero flux, branch 0
    f = oracle.face([0, 0, 0, 3, 1], [0, 0, 0, -2, 1])
    assert f["branch"] == 0 and f["Fm"] == f["Fn"] == f["Ft"] == 0


def test_hll_mirror_symmetry():
    """Mirroring x -> -x (swap L/R, negate normal velocity) negates the mass and transverse fluxes
    and preserves the normal-momentum flux, bit for bit."""
    rng = np.random.default_rng(4)
    for _ in range(500):
        hl, hr = rng.uniform(0, 2, 2)
        ul, ur, tl, tr = rng.normal(size=4) * 2
        f = oracle.face([hl, hl, 0, ul, tl], [hr, hr, 0, ur, tr])
        m = oracle.face([hr, hr, 0, -ur, tr], [hl, hl, 0, -ul, tl])
        assert m["Fm"] == -f["Fm"] and m["Fn"] == f["Fn"] and m["Ft"] == -f["Ft"]


def test_wall_face_zero_mass_flux():
    """A wall ghost = exact mirror (Q16): l = (h, eta, z, -u, t) against r = (h, eta, z, u, t) gives Fm = Ft = 0."""
    rng = np.random.default_rng(5)
    for _ in range(500):
        h = rng.uniform(0, 2)
        u, t = rng.normal(size=2)
        f = oracle.face([h, h, 0, -u, t], [h, h, 0, u, t])
        assert f["Fm"] == 0.0 and f["Ft"] == 0.0


def test_lake_at_rest_face_balance():
    """Lake at rest across a step: the flux + interface source equals g/2 h_face^2 on each side so that
    the well-balanced assembly cancels."""
    for zl, zr, eta in [(0.0, 0.3, 1.0), (0.5, 0.1, 0.8), (1.2, 0.0, 1.0)]:
        hl, hr = max(eta - zl, 0), max(eta - zr, 0)
        f = oracle.face([hl, eta if hl > 0 else zl, zl, 0, 0], [hr, eta if hr > 0 else zr, zr, 0, 0])
        assert f["Fm"] == 0.0
        assert abs((f["Fn"] + f["SL"]) - 0.5 * G * hl * hl) <= 1e-14
        assert abs((f["Fn"] + f["SR"]) - 0.5 * G * hr * hr) <= 1e-14


# ---------------------------------------------------------------- CFL
def test_cfl_single_cell():
    from workloads.configs import SwofConfig
    ex = SPEC["cfl"]
    cfg = SwofConfig(name="t", nx=1, ny=1, dx=ex["dx"], dy=ex["dx"], cfl=ex["n_cfl"])
    P = oracle.params_from_config(cfg)
    dt, ax, ay = oracle.cfl_dt(P, [[ex["h"]]], [[0.0]], [[0.0]])
    assert abs(2 * dt - ex["dt_prefix"]) < ex["prefix_tol"]
    # 1 cell: a_x = a_y = sqrt(g h); the 2D sum form (Q17) gives n_CFL/(2 a/dx), half the 1D value
    assert rel(2 * dt, ex["n_cfl"] * ex["dx"] / math.sqrt(G * ex["h"])) < 1e-15   # closed form
    # doubling dx doubles dt; all dry -> dt_max
    cfg2 = SwofConfig(name="t", nx=1, ny=1, dx=2 * ex["dx"], dy=2 * ex["dx"], cfl=ex["n_cfl"])
    assert oracle.cfl_dt(oracle.params_from_config(cfg2), [[1.0]], [[0.0]], [[0.0]])[0] == 2 * dt
    assert oracle.cfl_dt(P, [[0.0]], [[0.0]], [[0.0]])[0] == cfg.dt_max
    # t_end clip
    assert oracle.cfl_dt(P, [[1.0]], [[0.0]], [[0.0]], t=10.0, t_end=10.05)[0] == 10.05 - 10.0


# ---------------------------------------------------------------- friction
def test_friction_coefficients():
    ex = SPEC["manning_cf"]
    assert rel(oracle.friction_gcf("manning", ex["n"]) / G, ex["C_f"]) < 1e-15
    assert oracle.friction_gcf("strickler", 1.0) / G == 1.0
    ex = SPEC["darcy_cf"]
    assert rel(oracle.friction_gcf("darcy_weisbach", ex["f"]) / G, ex["C_f"]) < 1e-14
    # Chezy C_f = 1/C^2
    assert rel(oracle.friction_gcf("chezy", 50.0) / G, 1 / 2500) < 1e-15
    # Manning(n) and Strickler(K = 1/n) give the same coefficient
    assert rel(oracle.friction_gcf("strickler", 1 / 0.03), oracle.friction_gcf("manning", 0.03)) < 1e-15


def test_friction_darcy_example():
    ex = SPEC["friction_dw"]
    gcf = oracle.friction_gcf("darcy_weisbach", ex["f"])
    hu, hv = oracle.friction(gcf, "darcy_weisbach", ex["dt"], ex["h"], ex["q"], 0.0, ex["h"], ex["q"], 0.0)
    assert hu == ex["q_new"] and hv == 0.0


def test_friction_properties():
    rng = np.random.default_rng(6)
    for law in ("manning", "darcy_weisbach", "strickler", "chezy"):
        coef = {"manning": 0.04, "darcy_weisbach": 0.1, "strickler": 25.0, "chezy": 40.0}[law]
        gcf = oracle.friction_gcf(law, coef)
        for _ in range(200):
            hs, hst = rng.uniform(1e-3, 2, 2)
            hus, hvs, hup, hvp = rng.normal(size=4)
            a, b = oracle.friction(gcf, law, 0.1, hs, hus, hvs, hst, hup, hvp)
            # never increases |q|, never flips sign
            assert abs(a) <= abs(hup) and abs(b) <= abs(hvp)
            assert a * hup >= 0 and b * hvp >= 0
        # q^n = 0 -> unchanged; dry -> zero momentum; lake at rest stays at rest
        assert oracle.friction(gcf, law, 0.1, 1.0, 0.0, 0.0, 1.0, 0.3, -0.2) == (0.3, -0.2)
        assert oracle.friction(gcf, law, 0.1, 1.0, 1.0, 0.0, 1e-13, 0.3, -0.2) == (0.0, 0.0)
        assert oracle.friction(gcf, law, 0.1, 1.0, 0.0, 0.0, 1.0, 0.0, 0.0) == (0.0, 0.0)


def test_friction_manning_power():
    """Manning: q/(1 + dt g n^2 |u| / h^(4/3)) (P:82 with -g h S_f), checked against pow()."""
    rng = np.random.default_rng(7)
    gcf = oracle.friction_gcf("manning", 0.05)
    for _ in range(300):
        h = 10 ** rng.uniform(-6, 1.5)
        q = rng.normal()
        a, _ = oracle.friction(gcf, "manning", 0.2, h, q, 0.0, h, q, 0.0)
        want = q / (1 + 0.2 * G * 0.05 ** 2 * abs(q / h) / h ** (4.0 / 3.0))
        assert abs(a - want) <= 1e-14 * abs(want) + 1e-300


def test_friction_sheet_vs_printed_division():
    """DESIGN.md §3 Q11/Q20: the sheet evaluates the printed q* / (1 + w) as q* (1 / (1 + w)) -- one
    reciprocal for the two discharge components of a 2D cell.  Equal in exact arithmetic; in fp64 the two
    differ by at most 2 ulp (RN(1/d) then RN(q RN(1/d)) against the single RN(q/d)).  Pinned here against the
    printed division evaluated independently in numpy with the same w (Darcy/Chezy: w = k/h*; Manning/
    Strickler: w = k s^4 with s = icbrt(h*), icbrt itself pinned to libm cbrt in test_icbrt_accuracy)."""
    rng = np.random.default_rng(11)
    worst = 0.0
    for law, coef in (("darcy_weisbach", 0.05), ("chezy", 40.0), ("manning", 0.04), ("strickler", 25.0)):
        gcf = oracle.friction_gcf(law, coef)
        for _ in range(400):
            hs, hst = 10 ** rng.uniform(-4, 0.5, 2)
            hus, hvs, hup, hvp = rng.normal(size=4) * 0.5
            dt = rng.uniform(0.01, 1.0)
            a, b = oracle.friction(gcf, law, dt, hs, hus, hvs, hst, hup, hvp)
            umag = np.sqrt(hus * hus + hvs * hvs) * (1.0 / hs)
            k = (dt * gcf) * umag
            if law in ("darcy_weisbach", "chezy"):
                w = k / hst
            else:
                sg = oracle.icbrt(hst)
                w = k * ((sg * sg) * (sg * sg))
            for got, q in ((a, hup), (b, hvp)):
                want = q / (1.0 + w)             # the printed division
                ulp = np.spacing(abs(want))
                assert abs(got - want) <= 2 * ulp, (law, got, want)
                worst = max(worst, abs(got - want) / ulp)
    assert worst <= 2


# ---------------------------------------------------------------- icbrt (Q20)
def test_icbrt_accuracy():
    getcontext().prec = 50
    rng = np.random.default_rng(8)
    xs = list(10 ** rng.uniform(-14, 8, 2000)) + [1.0, 8.0, 27.0, 0.125, 2.0, 4.0, 0.5, 1e-12, 7.999999999]
    for x in xs:
        y = oracle.icbrt(x)
        # y^-3 should equal x: relative error of y within 2 ulp of the true x^(-1/3)
        err = abs(Decimal(y) ** 3 * Decimal(x) - 1)
        assert err < Decimal(3 * 2.3e-16), (x, y, err)
        # libm pow with the rounded exponent -1/3 differs from x^(-1/3) by ~|ln x| eps/3 itself
        assert abs(y - x ** (-1.0 / 3.0)) <= 1e-14 * y
        assert abs(1.0 / y - np.cbrt(x)) <= 4e-16 * np.cbrt(x) * 2
    assert oracle.icbrt(8.0) == 0.5 and oracle.icbrt(1.0) == 1.0 and oracle.icbrt(0.125) == 2.0


# ---------------------------------------------------------------- Green-Ampt
def _ga_params(Ks, A, hf, dtheta):
    from workloads.configs import SwofConfig, GreenAmpt
    cfg = SwofConfig(name="t", nx=1, ny=1, dx=1, dy=1, ga=GreenAmpt(Ks=Ks, hf=hf, A=A, dtheta=dtheta))
    return oracle.params_from_config(cfg)


def test_green_ampt_examples():
    ex = SPEC["ga_capacity"]
    P = _ga_params(ex["Ks"], ex["A"], ex["hf"], ex["dtheta"])
    # capacity at h_over -> 0 is 3e-5 m/s; with h_over = 3e-5 m the step is capacity-limited
    # and infiltrates Ks (A + (hf - h_over) dtheta / V) dt = 2.9994e-5 m (printed form, Q15)
    h, V = oracle.green_ampt(P, 3e-5, ex["V"], 1.0)
    inf = 3e-5 - h
    assert rel(inf, ex["I_C"]) < 3e-4 and rel(inf, 2.9994e-5) < 1e-9 and rel(V - ex["V"], inf) < 1e-9
    h, V = oracle.green_ampt(P, 1e-6, ex["V"], 1.0)    # supply-limited
    assert h == 0.0 and V == ex["V"] + 1e-6
    h, V = oracle.green_ampt(P, 0.0, ex["V"], 1.0)     # nothing to infiltrate
    assert h == 0.0 and V == ex["V"]
    Pz = _ga_params(0.0, 1.0, 0.1, 0.3)                # Ks = 0 -> impermeable
    assert oracle.green_ampt(Pz, 0.4, 0.01, 1.0) == (0.4, 0.01)
    # hf = h_over and A = 1 -> I_C = Ks
    P1 = _ga_params(2e-5, 1.0, 0.3, 0.3)
    h, V = oracle.green_ampt(P1, 0.3, 0.05, 2.0)
    assert rel(0.3 - h, 4e-5) < 1e-10
    # V = 0 -> unlimited capacity, all water infiltrates (Q15)
    assert oracle.green_ampt(P1, 0.25, 0.0, 1.0) == (0.0, 0.25)


def test_green_ampt_invariants():
    rng = np.random.default_rng(9)
    P = _ga_params(1e-5, 1.0, 0.1, 0.3)
    for _ in range(500):
        hr, V, dt = rng.uniform(0, 1e-3), rng.uniform(0, 0.05), rng.uniform(0.01, 2)
        h, V2 = oracle.green_ampt(P, hr, V, dt)
        assert 0.0 <= h <= hr and V2 >= V                      # I dt <= h_over, V non-decreasing
        assert abs((h + V2) - (hr + V)) <= 1e-15 * (hr + V)   # water moves from surface to soil


# ---------------------------------------------------------------- forcing tables
def test_rain_and_hydrograph_tables():
    from workloads.configs import SwofConfig, Inflow
    cfg = SwofConfig(name="t", nx=4, ny=4, dx=1, dy=1, rain_t=[0.0, 600.0], rain_rate=[1e-5, 0.0],
                     bc={"W": "inflow", "E": "free", "S": "wall", "N": "wall"},
                     inflow={"W": Inflow(0, 2, [0.0, 600.0], [50.0, 200.0])})
    P = oracle.params_from_config(cfg)
    assert oracle.rain_rate(P, -1.0) == 0.0 and oracle.rain_rate(P, 0.0) == 1e-5
    assert oracle.rain_rate(P, 599.999) == 1e-5 and oracle.rain_rate(P, 600.0) == 0.0   # [t_a, t_b)
    assert oracle.hydrograph(P, 0, 0.0) == 50.0 and oracle.hydrograph(P, 0, 300.0) == 125.0
    assert oracle.hydrograph(P, 0, 1e4) == 200.0


def test_pairwise_sum():
    x = np.arange(1, 1001, dtype=float)
    assert oracle.pairwise_sum(x) == 500500.0
    assert oracle.pairwise_sum(np.zeros(0)) == 0.0
