"""T4 for the scheme variants: Rusanov flux, first order + explicit Euler
(P:321), CFL on reconstructed values, Darcy-consistent Green-Ampt (Q15) -- the GPU (C ABI,
sm_100a kernels: the generic stage-kernel instance, the order-1 commit and the face-CFL pass) against
the oracle, element by element, with the tolerances of test_gpu_parity.py.
"""
import numpy as np
import pytest

import oracle
from swof_testlib import compare, gpu_run, gpu_solver
from test_gpu_parity import TOL_FULL, TOL_STEP, dt_close, masks_equal
from workloads import make

pytestmark = pytest.mark.gpu

VARIANTS = {
    "rusanov": dict(flux="rusanov"),
    "order1": dict(order=1, cfl=1.0),
    "cflface": dict(cfl_mode="face"),
    "darcyga": dict(ga_form="darcy"),
    "all": dict(flux="rusanov", order=1, cfl=1.0, cfl_mode="face", ga_form="darcy"),
    "dryskip": dict(dry_skip=True),          # GPU-only optimisation: results must not change
    # the other two friction laws of P:80-90 (C_f = 1/K^2 and 1/C^2); on cfg3 the per-cell field becomes
    # K = 1/n (resp. C = 1/n), so the kernels' per-cell branches of both laws run too
    "strickler": dict(fric_law="strickler", fric_coef=25.0),
    "chezy": dict(fric_law="chezy", fric_coef=40.0),
}
CASES = [("cfg0", 64, 64), ("cfg1", 100, 70), ("cfg3", 130, 90), ("cfg4", 75, 41)]


def variant_cfg(name, nx, ny, kw, steps):
    cfg = make(name, nx=nx, ny=ny)
    cfg.steps, cfg.t_end = steps, None
    for k, v in kw.items():
        setattr(cfg, k, v)
    if kw.get("fric_law") in ("strickler", "chezy") and cfg.fric_field is not None:
        cfg.fric_field = np.ascontiguousarray(1.0 / cfg.fric_field)
    if name == "cfg3":
        # the dry valley has no CFL speed, so step 0 takes dt = dt_max = 1 s while the critical inflow
        # ghost (Q18) pours in; the variants' corrector then clamps centimetres (both sides alike,
        # the clamp is part of the compared arithmetic): do not stop on it
        cfg.clamp_fail = 1.0
    return cfg


@pytest.mark.parametrize("vname", list(VARIANTS))
@pytest.mark.parametrize("name,nx,ny", CASES)
def test_variant_one_step(gpu, vname, name, nx, ny):
    cfg = variant_cfg(name, nx, ny, VARIANTS[vname], 1)
    g = gpu_run(cfg, nsteps=1)
    r = oracle.run(cfg)
    res = compare(g, r, TOL_STEP)
    dt_close(g["dt"], r["dt"])
    masks_equal(g, r)
    if cfg.ga is not None:
        assert np.max(np.abs(g["v"] - r["v"])) <= TOL_STEP
    print(vname, name, res)


@pytest.mark.parametrize("vname", list(VARIANTS))
@pytest.mark.parametrize("name,nx,ny", CASES)
def test_variant_many_steps(gpu, vname, name, nx, ny):
    cfg = variant_cfg(name, nx, ny, VARIANTS[vname], 150)
    g = gpu_run(cfg, nsteps=150, graph_steps=8)
    r = oracle.run(cfg)
    assert g["step"] == r["steps"] == 150
    res = compare(g, r, TOL_FULL)
    dt_close(g["dt"], r["dt"])
    masks_equal(g, r)
    if cfg.ga is not None:
        assert np.max(np.abs(g["v"] - r["v"])) <= TOL_FULL
    assert g["diag"]["flags"] == 0
    print(vname, name, res)


@pytest.mark.parametrize("vname", ["order1", "cflface"])
def test_variant_run_to_t_end(gpu, vname):
    """swof_run with the variant's step protocol: lands on t_end exactly, no-op steps past it."""
    cfg = variant_cfg("cfg2", 97, 53, VARIANTS[vname], None)
    cfg.steps, cfg.t_end = None, 120.0
    g = gpu_run(cfg, t_end=cfg.t_end)
    r = oracle.run(cfg)
    assert g["t"] == r["t"] == 120.0 and g["step"] == r["steps"]
    compare(g, r, TOL_FULL)
    dt_close(g["dt"], r["dt"])
    s = gpu_solver(cfg)
    s.run(cfg.t_end)
    a = s.get_state()
    assert s.run(cfg.t_end) == 0                 # t >= t_end: nothing to do
    b = s.get_state()
    s.close()
    assert b["step"] == a["step"] and all(np.array_equal(a[k], b[k]) for k in ("h", "hu", "hv"))


def test_order1_predictor_is_the_step(gpu):
    cfg = variant_cfg("cfg4", 75, 41, VARIANTS["order1"], 1)
    s = gpu_solver(cfg)
    p = s.predictor()
    s.step(1)
    st = s.get_state()
    s.close()
    assert all(np.array_equal(p[k], st[k]) for k in ("h", "hu", "hv"))


def test_variant_launch_counts(gpu):
    for vname, n in (("rusanov", 2), ("order1", 2), ("cflface", 3), ("all", 3)):
        s = gpu_solver(variant_cfg("cfg0", 64, 64, VARIANTS[vname], 1))
        assert s.launches_per_step() == n, vname
        s.close()


@pytest.mark.parametrize("name,nx,ny", [("cfg2", 97, 53), ("cfg3", 130, 90)])
def test_dry_skip_on_drying_domains(gpu, name, nx, ny):
    """Mostly dry domains (rain infiltrating, an inflow front): the all-dry tiles take the skip path."""
    cfg = make(name, nx=nx, ny=ny)
    cfg.steps, cfg.t_end = 200, None
    base = gpu_run(cfg, nsteps=200)
    cfg.dry_skip = True
    fast = gpu_run(cfg, nsteps=200)
    for k in ("h", "hu", "hv", "v"):
        assert np.array_equal(fast[k], base[k]), k
    assert np.array_equal(fast["dt"], base["dt"])
    r = oracle.run(cfg)
    compare(fast, r, TOL_FULL)
