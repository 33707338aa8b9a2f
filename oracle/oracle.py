"""ctypes binding of oracle/swof_oracle.c (TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py).

Argument marshalling only: every arithmetic step of the oracle is in the C file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "swof_oracle.c"
_HDR = _HERE / "swof_oracle.h"
_LIB = _HERE / "liboracle.so"
_LIB_OMP = _HERE / "liboracle_omp.so"      # OpenMP-over-rows build (bitwise identical; development aid)
# -ffp-contract=off: no FMA contraction; no -march=native, no -ffast-math (IEEE div/sqrt)
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]

MAXT = 16
FRIC = {"none": 0, "manning": 1, "strickler": 2, "darcy_weisbach": 3, "chezy": 4}
BC = {"wall": 0, "free": 1, "periodic": 2, "inflow": 3}
SIDES = ("W", "E", "S", "N")


class OrParams(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("dx", C.c_double), ("dy", C.c_double),
        ("g", C.c_double), ("cfl", C.c_double), ("dt_max", C.c_double), ("h_eps", C.c_double),
        ("fric_law", C.c_int32), ("fric_coef", C.c_double),
        ("ga_enabled", C.c_int32), ("ga_Ks", C.c_double), ("ga_hf", C.c_double), ("ga_A", C.c_double),
        ("ga_dtheta", C.c_double), ("ga_vinf0", C.c_double),
        ("n_rain", C.c_int32), ("rain_t", C.c_double * MAXT), ("rain_rate", C.c_double * MAXT),
        ("bc", C.c_int32 * 4), ("in_k0", C.c_int32 * 4), ("in_k1", C.c_int32 * 4), ("n_hydro", C.c_int32 * 4),
        ("hydro_t", (C.c_double * MAXT) * 4), ("hydro_q", (C.c_double * MAXT) * 4),
        ("flux", C.c_int32), ("order", C.c_int32), ("cfl_mode", C.c_int32), ("ga_form", C.c_int32),
    ]


FLUX = {"hll": 0, "rusanov": 1}
CFL_MODE = {"cell": 0, "face": 1}
GA_FORM = {"printed": 0, "darcy": 1}


class Counters(C.Structure):
    _fields_ = [("face_dry", C.c_int64), ("face_left", C.c_int64), ("face_right", C.c_int64),
                ("face_mid", C.c_int64), ("cell_stage", C.c_int64), ("cell_wet_fric", C.c_int64),
                ("ga_capped", C.c_int64), ("clamps", C.c_int64), ("clamped_mass", C.c_double),
                ("clamp_max", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def build(force: bool = False, omp: bool = False) -> Path:
    """Compile liboracle.so (or, omp=True, liboracle_omp.so with -fopenmp) with gcc (building the checker is
    not using it)."""
    out = _LIB_OMP if omp else _LIB
    if not force and out.exists() and out.stat().st_mtime >= max(_SRC.stat().st_mtime, _HDR.stat().st_mtime):
        return out
    tmp = out.with_suffix(f".so.tmp{os.getpid()}")
    subprocess.run(["gcc", *CFLAGS, *(["-fopenmp"] if omp else []), "-o", str(tmp), str(_SRC), "-lm"], check=True)
    os.replace(tmp, out)
    return out


_lib = None
_lib_omp = None
_D = C.POINTER(C.c_double)


def lib(omp: bool = False):
    """The oracle library; omp=True: the OpenMP-over-rows build (same results bit for bit)."""
    global _lib, _lib_omp
    if omp:
        if _lib_omp is None:
            _lib_omp = _declare(C.CDLL(str(build(omp=True))))
        return _lib_omp
    if _lib is None:
        _lib = _declare(C.CDLL(str(build())))
    return _lib


def _declare(L):
    if True:
        P = C.POINTER(OrParams)
        L.or_minmod.restype = C.c_double
        L.or_minmod.argtypes = [C.c_double, C.c_double]
        L.or_icbrt.restype = C.c_double
        L.or_icbrt.argtypes = [C.c_double]
        L.or_rain_rate.restype = C.c_double
        L.or_rain_rate.argtypes = [P, C.c_double]
        L.or_hydrograph.restype = C.c_double
        L.or_hydrograph.argtypes = [P, C.c_int, C.c_double]
        L.or_friction_gcf.restype = C.c_double
        L.or_friction_gcf.argtypes = [C.c_int, C.c_double, C.c_double]
        L.or_muscl_cell.restype = None
        L.or_muscl_cell.argtypes = [_D, _D, _D, _D, C.c_double, _D]
        L.or_centered_source.restype = C.c_double
        L.or_centered_source.argtypes = [C.c_double] * 5
        L.or_face.restype = C.c_int
        L.or_face.argtypes = [C.c_double, C.c_double, _D, _D, _D]
        L.or_face_rusanov.restype = C.c_int
        L.or_face_rusanov.argtypes = [C.c_double, C.c_double, _D, _D, _D]
        L.or_cfl_dt_face.restype = C.c_double
        L.or_cfl_dt_face.argtypes = [P, _D, _D, _D, _D, C.c_double, C.c_double, C.c_double, _D, _D]
        L.or_green_ampt.restype = None
        L.or_green_ampt.argtypes = [P, C.c_double, C.c_double, C.c_double, _D, _D]
        L.or_friction.restype = None
        L.or_friction.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_double, C.c_double, _D, _D]
        L.or_cfl_dt.restype = C.c_double
        L.or_cfl_dt.argtypes = [P, _D, _D, _D, C.c_double, C.c_double, _D, _D]
        L.or_stage.restype = C.c_int
        L.or_stage.argtypes = [P, _D, _D, _D, _D, _D, _D, C.c_double, C.c_double, _D, _D, _D, _D,
                               C.POINTER(Counters)]
        L.or_heun_step.restype = C.c_int
        L.or_heun_step.argtypes = [P, _D, _D, _D, _D, _D, _D, C.c_double, C.c_double, C.POINTER(Counters)]
        L.or_run.restype = C.c_int
        L.or_run.argtypes = [P, _D, _D, _D, _D, _D, _D, _D, C.c_int64, C.c_double, C.c_double, _D,
                             C.c_int64, C.POINTER(C.c_int64), C.POINTER(Counters)]
        L.or_flow_direction.restype = None
        L.or_flow_direction.argtypes = [_D, C.c_int32, C.c_int32, C.c_void_p]
        L.or_flow_direction_f32.restype = None
        L.or_flow_direction_f32.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]
        L.or_pairwise_sum.restype = C.c_double
        L.or_pairwise_sum.argtypes = [_D, C.c_int64]
    return L


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _arr(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def params_from_config(cfg) -> OrParams:
    """workloads.SwofConfig -> OrParams (the oracle's own parameter struct)."""
    P = OrParams()
    P.nx, P.ny, P.dx, P.dy = cfg.nx, cfg.ny, cfg.dx, cfg.dy
    P.g, P.cfl, P.dt_max, P.h_eps = cfg.g, cfg.cfl, cfg.dt_max, cfg.h_eps
    P.fric_law, P.fric_coef = FRIC[cfg.fric_law], cfg.fric_coef
    if cfg.ga is not None:
        P.ga_enabled = 1
        P.ga_Ks, P.ga_hf, P.ga_A, P.ga_dtheta, P.ga_vinf0 = (cfg.ga.Ks, cfg.ga.hf, cfg.ga.A, cfg.ga.dtheta,
                                                            cfg.ga.vinf0)
    P.n_rain = len(cfg.rain_rate)
    for k, (t, r) in enumerate(zip(cfg.rain_t, cfg.rain_rate)):
        P.rain_t[k], P.rain_rate[k] = t, r
    for s, side in enumerate(SIDES):
        P.bc[s] = BC[cfg.bc[side]]
        if side in cfg.inflow:
            fl = cfg.inflow[side]
            P.in_k0[s], P.in_k1[s] = fl.k0, fl.k1
            P.n_hydro[s] = len(fl.hydro_t)
            for k, (t, q) in enumerate(zip(fl.hydro_t, fl.hydro_q)):
                P.hydro_t[s][k], P.hydro_q[s][k] = t, q
    P.flux = FLUX[getattr(cfg, "flux", "hll")]
    P.order = int(getattr(cfg, "order", 2))
    P.cfl_mode = CFL_MODE[getattr(cfg, "cfl_mode", "cell")]
    P.ga_form = GA_FORM[getattr(cfg, "ga_form", "printed")]
    return P


# ---- pointwise wrappers -----------------------------------------------------------------------
def minmod(a, b):
    return lib().or_minmod(a, b)


def icbrt(x):
    return lib().or_icbrt(x)


def rain_rate(P, t):
    return lib().or_rain_rate(C.byref(P), t)


def hydrograph(P, side, t):
    return lib().or_hydrograph(C.byref(P), side, t)


def friction_gcf(law, coef, g=9.81):
    return lib().or_friction_gcf(FRIC[law] if isinstance(law, str) else law, coef, g)


def muscl_cell(h3, eta3, u3, v3, rh_c):
    out = np.zeros(10)
    lib().or_muscl_cell(_p(_arr(h3)), _p(_arr(eta3)), _p(_arr(u3)), _p(_arr(v3)), rh_c, _p(out))
    return dict(zip(("hm", "hp", "em", "ep", "zm", "zp", "um", "up", "vm", "vp"), out))


def centered_source(hm, hp, zm, zp, g=9.81):
    return lib().or_centered_source(g, hm, hp, zm, zp)


def face(l, r, g=9.81, h_eps=1e-12):
    """l, r = (h, eta, z, u_normal, u_transverse) of the left cell's high face / right cell's low face."""
    out = np.zeros(9)
    br = lib().or_face(g, h_eps, _p(_arr(l)), _p(_arr(r)), _p(out))
    d = dict(zip(("Fm", "Fn", "Ft", "SL", "SR", "HL", "HR", "c1", "c2"), out))
    d["branch"] = br
    return d


def face_rusanov(l, r, g=9.81, h_eps=1e-12):
    """Rusanov face: same inputs as face(); out c = the wave-speed bound."""
    out = np.zeros(9)
    br = lib().or_face_rusanov(g, h_eps, _p(_arr(l)), _p(_arr(r)), _p(out))
    d = dict(zip(("Fm", "Fn", "Ft", "SL", "SR", "HL", "HR", "c", "_"), out))
    d["branch"] = br
    return d


def green_ampt(P, h_r, V, dt):
    ho, vo = C.c_double(), C.c_double()
    lib().or_green_ampt(C.byref(P), h_r, V, dt, C.byref(ho), C.byref(vo))
    return ho.value, vo.value


def friction(gcf, law, dt, hs, hus, hvs, hst, hup, hvp, h_eps=1e-12):
    a, b = C.c_double(), C.c_double()
    lib().or_friction(gcf, FRIC[law] if isinstance(law, str) else law, h_eps, dt, hs, hus, hvs, hst, hup, hvp,
                      C.byref(a), C.byref(b))
    return a.value, b.value


def flow_direction(z):
    """D8 flow direction (listing P:683-708) of a (ny, nx) DEM, float64 or float32 -> uint8 0..8."""
    z = np.ascontiguousarray(z)
    ny, nx = z.shape
    out = np.empty((ny, nx), dtype=np.uint8)
    if z.dtype == np.float32:
        lib().or_flow_direction_f32(C.c_void_p(z.ctypes.data), nx, ny, C.c_void_p(out.ctypes.data))
    else:
        z = _arr(z)
        lib().or_flow_direction(_p(z), nx, ny, C.c_void_p(out.ctypes.data))
    return out


def pairwise_sum(x):
    x = _arr(x).ravel()
    return lib().or_pairwise_sum(_p(x), x.size)


# ---- whole-array wrappers ---------------------------------------------------------------------
def cfl_dt(P, h, hu, hv, t=0.0, t_end=float("inf")):
    ax, ay = C.c_double(), C.c_double()
    dt = lib().or_cfl_dt(C.byref(P), _p(_arr(h)), _p(_arr(hu)), _p(_arr(hv)), t, t_end, C.byref(ax), C.byref(ay))
    return dt, ax.value, ay.value


def cfl_dt_face(P, z, h, hu, hv, t_ghost=0.0, t=0.0, t_end=float("inf")):
    ax, ay = C.c_double(), C.c_double()
    dt = lib().or_cfl_dt_face(C.byref(P), _p(_arr(z)), _p(_arr(h)), _p(_arr(hu)), _p(_arr(hv)), t_ghost, t, t_end,
                              C.byref(ax), C.byref(ay))
    return dt, ax.value, ay.value


def stage(P, z, fric, h, hu, hv, v, t_s, dt):
    h, hu, hv, z = _arr(h), _arr(hu), _arr(hv), _arr(z)
    v = _arr(v) if v is not None else None
    fric = _arr(fric) if fric is not None else None
    oh, ohu, ohv = np.empty_like(h), np.empty_like(h), np.empty_like(h)
    ov = np.empty_like(h) if v is not None else None
    cnt = Counters()
    rc = lib().or_stage(C.byref(P), _p(z), _p(fric), _p(h), _p(hu), _p(hv), _p(v), t_s, dt,
                        _p(oh), _p(ohu), _p(ohv), _p(ov), C.byref(cnt))
    if rc:
        raise RuntimeError(f"or_stage failed: {rc}")
    return oh, ohu, ohv, ov, cnt


def heun_step(P, z, fric, h, hu, hv, v, t, dt):
    h, hu, hv = _arr(h).copy(), _arr(hu).copy(), _arr(hv).copy()
    v = _arr(v).copy() if v is not None else None
    cnt = Counters()
    rc = lib().or_heun_step(C.byref(P), _p(_arr(z)), _p(_arr(fric) if fric is not None else None),
                            _p(h), _p(hu), _p(hv), _p(v), t, dt, C.byref(cnt))
    if rc:
        raise RuntimeError(f"or_heun_step failed: {rc}")
    return h, hu, hv, v, cnt


def run(cfg_or_P, z=None, fric=None, h=None, hu=None, hv=None, v=None, t0=0.0, nsteps=None,
        t_end=float("inf"), dt_forced=0.0, omp=False):
    """Run the oracle time loop.  Accepts a workloads.SwofConfig (inputs taken from it) or OrParams.
    omp=True runs the OpenMP-over-rows build (bitwise identical state; counters summed in another order)."""
    if isinstance(cfg_or_P, OrParams):
        P = cfg_or_P
    else:
        cfg = cfg_or_P
        P = params_from_config(cfg)
        z = cfg.z if z is None else z
        fric = cfg.fric_field if fric is None else fric
        h = cfg.h if h is None else h
        hu = cfg.hu if hu is None else hu
        hv = cfg.hv if hv is None else hv
        if v is None and cfg.ga is not None:
            v = cfg.vinf if cfg.vinf is not None else np.full((cfg.ny, cfg.nx), cfg.ga.vinf0)
        if nsteps is None:
            nsteps = cfg.steps if cfg.steps is not None else 1 << 40
        if cfg.t_end is not None and t_end == float("inf"):
            t_end = cfg.t_end
    h, hu, hv = _arr(h).copy(), _arr(hu).copy(), _arr(hv).copy()
    v = _arr(v).copy() if (v is not None and P.ga_enabled) else None
    cap = int(min(nsteps, 1 << 22))
    dth = np.zeros(cap)
    t = C.c_double(t0)
    done = C.c_int64()
    cnt = Counters()
    rc = lib(omp).or_run(C.byref(P), _p(_arr(z)), _p(_arr(fric) if fric is not None else None),
                      _p(h), _p(hu), _p(hv), _p(v), C.byref(t), int(nsteps), t_end, dt_forced,
                      _p(dth), cap, C.byref(done), C.byref(cnt))
    return {"rc": rc, "h": h, "hu": hu, "hv": hv, "v": v, "t": t.value, "steps": done.value,
            "dt": dth[: min(done.value, cap)], "counters": cnt}
