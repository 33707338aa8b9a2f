"""Thin ctypes binding of libswof.so (include/swof.h): argument marshalling only.

Every step of the time loop runs in the CUDA kernels of csrc/; there is no CPU path.  PyTorch is used
only for device memory (the workspace) and the CUDA stream.  Importing this module without the
built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

# SWOF_LIB: an alternative build of the same library (tests: the bounds-checked -DSWOF_CHECK=1 build)
_LIB_PATH = Path(os.environ.get("SWOF_LIB", Path(__file__).resolve().parent / "libswof.so"))

SWOF_OK, SWOF_EINVAL, SWOF_ENUMERIC, SWOF_ECUDA, SWOF_ENOMEM, SWOF_ESTATE = range(6)
FRIC = {"none": 0, "manning": 1, "strickler": 2, "darcy_weisbach": 3, "chezy": 4}
BC = {"wall": 0, "free": 1, "periodic": 2, "inflow": 3, "halo": 4}
FLUX = {"hll": 0, "rusanov": 1}
CFL_MODE = {"cell": 0, "face": 1}
GA_FORM = {"printed": 0, "darcy": 1}
SIDES = ("W", "E", "S", "N")
MAXT = 16
FLAG_NONFINITE, FLAG_BIGCLAMP, FLAG_BADINPUT = 1, 2, 4
EXPORTS = ("swof_workspace_size", "swof_create", "swof_set_state", "swof_step", "swof_run", "swof_get_state",
           "swof_get_dt_history", "swof_get_diag", "swof_predictor", "swof_step_profiled",
           "swof_launches_per_step", "swof_ctx_launches_per_step", "swof_selftest_math", "swof_destroy",
           "swof_last_error", "swof_strerror", "swof_flow_direction", "swof_flow_direction_f32",
           "swof_halo_rows", "swof_enqueue_phase", "swof_cfl_maxima", "swof_refresh_cfl", "swof_set_limits",
           "swof_sync", "swof_set_halo_push", "swof_ipc_handle", "swof_ipc_open", "swof_ipc_close",
           "swof_copy", "swof_check_line")
SIDE_S, SIDE_N = 2, 3


class SwofParams(C.Structure):
    """Mirror of `swof_params` (include/swof.h)."""
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("dx", C.c_double), ("dy", C.c_double),
        ("g", C.c_double), ("cfl", C.c_double), ("dt_max", C.c_double), ("h_eps", C.c_double),
        ("fric_law", C.c_int32), ("fric_coef", C.c_double),
        ("ga_enabled", C.c_int32), ("ga_Ks", C.c_double), ("ga_hf", C.c_double), ("ga_A", C.c_double),
        ("ga_dtheta", C.c_double), ("ga_vinf0", C.c_double),
        ("n_rain", C.c_int32), ("rain_t", C.c_double * MAXT), ("rain_rate", C.c_double * MAXT),
        ("bc", C.c_int32 * 4), ("inflow_k0", C.c_int32 * 4), ("inflow_k1", C.c_int32 * 4),
        ("n_hydro", C.c_int32 * 4), ("hydro_t", (C.c_double * MAXT) * 4), ("hydro_q", (C.c_double * MAXT) * 4),
        ("dt_hist_cap", C.c_int64), ("graph_steps", C.c_int32), ("clamp_fail", C.c_double),
        ("flux", C.c_int32), ("order", C.c_int32), ("cfl_mode", C.c_int32), ("ga_form", C.c_int32),
        ("inflow_width", C.c_double * 4), ("dry_skip", C.c_int32),
    ]


class SwofDiag(C.Structure):
    """Mirror of `swof_diag` (include/swof.h)."""
    _fields_ = [("t", C.c_double), ("step", C.c_int64), ("dt_next", C.c_double), ("volume", C.c_double),
                ("vinf_volume", C.c_double), ("h_min", C.c_double), ("h_max", C.c_double),
                ("wet_cells", C.c_int64), ("clamps", C.c_int64), ("clamped_mass", C.c_double),
                ("clamp_max", C.c_double), ("flags", C.c_uint32),
                ("big_clamp_cell", C.c_int64), ("big_clamp_step", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class SwofError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"swof error {code}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load libswof.so; raises if it is missing (no fallback of any kind)."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(f"{_LIB_PATH} not built: run `python -m paper_1307_4839_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(str(_LIB_PATH))
        vp, dp, i64p = C.c_void_p, C.c_void_p, C.POINTER(C.c_int64)
        PP = C.POINTER(SwofParams)
        L.swof_workspace_size.argtypes = [PP, C.POINTER(C.c_size_t)]
        L.swof_create.argtypes = [PP, dp, dp, vp, C.c_size_t, vp, C.POINTER(C.c_void_p)]
        L.swof_set_state.argtypes = [vp, dp, dp, dp, dp, C.c_double]
        L.swof_step.argtypes = [vp, C.c_int64]
        L.swof_run.argtypes = [vp, C.c_double, C.c_int64, i64p]
        L.swof_get_state.argtypes = [vp, dp, dp, dp, dp, C.POINTER(C.c_double), i64p]
        L.swof_get_dt_history.argtypes = [vp, dp, C.c_int64, i64p]
        L.swof_get_diag.argtypes = [vp, C.POINTER(SwofDiag)]
        L.swof_predictor.argtypes = [vp, dp, dp, dp, dp]
        L.swof_step_profiled.argtypes = [vp, C.c_int64, C.POINTER(C.c_double)]
        L.swof_launches_per_step.argtypes = []
        L.swof_ctx_launches_per_step.argtypes = [vp]
        L.swof_selftest_math.argtypes = [C.c_int64, C.c_uint64, C.POINTER(C.c_int64)]
        L.swof_flow_direction.argtypes = [vp, C.c_int32, C.c_int32, vp, vp]
        L.swof_flow_direction_f32.argtypes = [vp, C.c_int32, C.c_int32, vp, vp]
        PD = C.POINTER(C.c_void_p)
        L.swof_halo_rows.argtypes = [vp, C.c_int32, C.c_int32, PD, PD, C.POINTER(C.c_size_t)]
        L.swof_enqueue_phase.argtypes = [vp, C.c_int32]
        L.swof_cfl_maxima.argtypes = [vp, PD]
        L.swof_refresh_cfl.argtypes = [vp]
        L.swof_set_limits.argtypes = [vp, C.c_double, C.c_int64]
        L.swof_sync.argtypes = [vp]
        L.swof_set_halo_push.argtypes = [vp, C.c_int32, PD, PD]
        L.swof_ipc_handle.argtypes = [vp, vp, C.POINTER(C.c_uint64)]
        L.swof_ipc_open.argtypes = [vp, PD]
        L.swof_ipc_close.argtypes = [vp]
        L.swof_copy.argtypes = [vp, vp, C.c_size_t, vp]
        L.swof_check_line.argtypes = []
        L.swof_destroy.argtypes = [vp]
        L.swof_destroy.restype = None
        L.swof_last_error.argtypes = [vp]
        L.swof_last_error.restype = C.c_char_p
        L.swof_strerror.argtypes = [C.c_int]
        L.swof_strerror.restype = C.c_char_p
        for name in ("swof_workspace_size", "swof_create", "swof_set_state", "swof_step", "swof_run",
                     "swof_get_state", "swof_get_dt_history", "swof_get_diag", "swof_predictor",
                     "swof_step_profiled", "swof_launches_per_step", "swof_ctx_launches_per_step",
                     "swof_selftest_math", "swof_flow_direction", "swof_flow_direction_f32", "swof_halo_rows",
                     "swof_enqueue_phase", "swof_cfl_maxima", "swof_refresh_cfl", "swof_set_limits", "swof_sync",
                     "swof_set_halo_push", "swof_ipc_handle", "swof_ipc_open", "swof_ipc_close", "swof_copy",
                     "swof_check_line"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def params_from_config(cfg, graph_steps: int = 0, dt_hist_cap: int = 0) -> SwofParams:
    """Problem statement (a workloads.SwofConfig or any object with the same attributes) -> swof_params."""
    p = SwofParams()
    p.nx, p.ny, p.dx, p.dy = cfg.nx, cfg.ny, cfg.dx, cfg.dy
    p.g, p.cfl, p.dt_max, p.h_eps = cfg.g, cfg.cfl, cfg.dt_max, cfg.h_eps
    p.fric_law, p.fric_coef = FRIC[cfg.fric_law], cfg.fric_coef
    if cfg.ga is not None:
        p.ga_enabled = 1
        p.ga_Ks, p.ga_hf, p.ga_A, p.ga_dtheta, p.ga_vinf0 = cfg.ga.Ks, cfg.ga.hf, cfg.ga.A, cfg.ga.dtheta, cfg.ga.vinf0
    p.n_rain = len(cfg.rain_rate)
    for k, (t, r) in enumerate(zip(cfg.rain_t, cfg.rain_rate)):
        p.rain_t[k], p.rain_rate[k] = t, r
    for s, side in enumerate(SIDES):
        p.bc[s] = BC[cfg.bc[side]]
        fl = cfg.inflow.get(side) if cfg.inflow else None
        if fl is not None:
            p.inflow_k0[s], p.inflow_k1[s] = fl.k0, fl.k1
            p.n_hydro[s] = len(fl.hydro_t)
            for k, (t, q) in enumerate(zip(fl.hydro_t, fl.hydro_q)):
                p.hydro_t[s][k], p.hydro_q[s][k] = t, q
            p.inflow_width[s] = float(getattr(fl, "width", 0.0) or 0.0)
    p.dt_hist_cap = dt_hist_cap
    p.graph_steps = graph_steps
    p.flux = FLUX[getattr(cfg, "flux", "hll")]
    p.order = int(getattr(cfg, "order", 2))
    p.cfl_mode = CFL_MODE[getattr(cfg, "cfl_mode", "cell")]
    p.ga_form = GA_FORM[getattr(cfg, "ga_form", "printed")]
    p.clamp_fail = float(getattr(cfg, "clamp_fail", 0.0))
    p.dry_skip = int(bool(getattr(cfg, "dry_skip", False)))
    return p


def _ptr(a, shape):
    """Host numpy array or torch tensor (host or CUDA) -> raw pointer; fp64, C-contiguous, (ny, nx)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):                       # torch.Tensor
        import torch
        assert a.dtype == torch.float64 and a.is_contiguous() and tuple(a.shape) == shape, (a.dtype, a.shape)
        return C.c_void_p(a.data_ptr())
    assert isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.shape == shape, \
        (type(a), getattr(a, "dtype", None), getattr(a, "shape", None))
    return C.c_void_p(a.ctypes.data)


class Solver:
    """One swof_ctx: a grid advanced on one GPU.  `stream`: a torch.cuda.Stream (default: current)."""

    def __init__(self, params: SwofParams, z, fric_field=None, stream=None, use_torch_workspace: bool = True,
                 device=None):
        import torch
        self._L = lib()
        self.params = params
        self.shape = (params.ny, params.nx)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        with torch.cuda.device(self.device):
            self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
            nbytes = C.c_size_t()
            self._check(self._L.swof_workspace_size(C.byref(params), C.byref(nbytes)), None)
            self.workspace_bytes = nbytes.value
            self._ws = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device) if use_torch_workspace else None
            ctx = C.c_void_p()
            rc = self._L.swof_create(C.byref(params), _ptr(z, self.shape), _ptr(fric_field, self.shape),
                                     C.c_void_p(self._ws.data_ptr()) if self._ws is not None else None,
                                     nbytes.value, C.c_void_p(self.stream.cuda_stream), C.byref(ctx))
            if rc != SWOF_OK:
                raise SwofError(rc, self._L.swof_strerror(rc).decode())
            self._ctx = ctx

    # -- helpers
    def _check(self, rc, ctx=None):
        if rc != SWOF_OK:
            msg = self._L.swof_last_error(ctx if ctx is not None else getattr(self, "_ctx", None)).decode() \
                if (ctx is not None or getattr(self, "_ctx", None)) else self._L.swof_strerror(rc).decode()
            raise SwofError(rc, msg)
        return rc

    def close(self):
        if getattr(self, "_ctx", None):
            self._L.swof_destroy(self._ctx)
            self._ctx = None
        self._ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- API (names follow include/swof.h)
    def set_state(self, h, hu, hv, v_inf=None, t0: float = 0.0):
        self._check(self._L.swof_set_state(self._ctx, _ptr(h, self.shape), _ptr(hu, self.shape), _ptr(hv, self.shape),
                                           _ptr(v_inf, self.shape), float(t0)))

    def step(self, nsteps: int):
        self._check(self._L.swof_step(self._ctx, int(nsteps)))

    def run(self, t_end: float, max_steps: int = 1 << 62) -> int:
        n = C.c_int64()
        self._check(self._L.swof_run(self._ctx, float(t_end), int(max_steps), C.byref(n)))
        return n.value

    def get_state(self, h=None, hu=None, hv=None, v_inf=None):
        """Copy the state into the given arrays (numpy or torch, host or device); allocates numpy if None."""
        out = {}
        for k, a in (("h", h), ("hu", hu), ("hv", hv), ("v", v_inf)):
            if a is None and (k != "v" or self.params.ga_enabled):
                a = np.empty(self.shape)
            out[k] = a
        t, s = C.c_double(), C.c_int64()
        self._check(self._L.swof_get_state(self._ctx, _ptr(out["h"], self.shape), _ptr(out["hu"], self.shape),
                                           _ptr(out["hv"], self.shape), _ptr(out["v"], self.shape),
                                           C.byref(t), C.byref(s)))
        out["t"], out["step"] = t.value, s.value
        return out

    def predictor(self):
        out = {k: np.empty(self.shape) for k in ("h", "hu", "hv")}
        out["v"] = np.empty(self.shape) if self.params.ga_enabled else None
        self._check(self._L.swof_predictor(self._ctx, _ptr(out["h"], self.shape), _ptr(out["hu"], self.shape),
                                           _ptr(out["hv"], self.shape), _ptr(out["v"], self.shape)))
        return out

    def dt_history(self, cap: int = 1 << 22):
        d = self.diag()
        cap = min(cap, d["step"])
        buf = np.empty(max(cap, 1))
        n = C.c_int64()
        self._check(self._L.swof_get_dt_history(self._ctx, C.c_void_p(buf.ctypes.data), cap, C.byref(n)))
        return buf[: n.value]

    def diag(self):
        d = SwofDiag()
        self._check(self._L.swof_get_diag(self._ctx, C.byref(d)))
        return d.as_dict()

    def step_profiled(self, nsteps: int):
        ms = (C.c_double * 2)()
        self._check(self._L.swof_step_profiled(self._ctx, int(nsteps), ms))
        return ms[0], ms[1]

    # -- row-strip decomposition support (include/swof.h, SWOF_BC_HALO)
    def _view(self, ptr: int, nbytes: int, dtype):
        """torch view of `nbytes` of this context's workspace starting at device address `ptr`."""
        assert self._ws is not None, "strip views need the torch workspace"
        off = ptr - self._ws.data_ptr()
        assert 0 <= off and off + nbytes <= self._ws.numel()
        return self._ws[off: off + nbytes].view(dtype)

    def halo_rows(self, field_set: int, side: int):
        """([send views], [recv views]) of the 2-row blocks of field set 0 (U^n), 1 (U*) or 2 (z)."""
        import torch
        send, recv = (C.c_void_p * 3)(), (C.c_void_p * 3)()
        nb = C.c_size_t()
        self._check(self._L.swof_halo_rows(self._ctx, field_set, side, send, recv, C.byref(nb)))
        sv = [self._view(send[k], nb.value, torch.float64) for k in range(3) if send[k]]
        rv = [self._view(recv[k], nb.value, torch.float64) for k in range(3) if recv[k]]
        return sv, rv

    def set_halo_push(self, side: int, set0_ptrs, set1_ptrs):
        """Fused exchange: device addresses (ints) of the neighbour's 3 receive blocks per field set."""
        a = (C.c_void_p * 3)(*set0_ptrs) if set0_ptrs is not None else None
        b = (C.c_void_p * 3)(*set1_ptrs) if set1_ptrs is not None else None
        self._check(self._L.swof_set_halo_push(self._ctx, side, a, b))

    def ipc_handle(self):
        """(64-byte IPC handle of the library-allocated workspace, its base address here)."""
        h = (C.c_ubyte * 64)()
        base = C.c_uint64()
        self._check(self._L.swof_ipc_handle(self._ctx, h, C.byref(base)))
        return bytes(h), base.value

    def halo_block_addrs(self, field_set: int, side: int):
        """Device addresses ([send x3], [recv x3]) of the 2-row blocks (see halo_rows)."""
        send, recv = (C.c_void_p * 3)(), (C.c_void_p * 3)()
        nb = C.c_size_t()
        self._check(self._L.swof_halo_rows(self._ctx, field_set, side, send, recv, C.byref(nb)))
        return [send[k] for k in range(3)], [recv[k] for k in range(3)], nb.value

    def enqueue_phase(self, phase: int):
        self._check(self._L.swof_enqueue_phase(self._ctx, phase))

    def cfl_maxima(self):
        """int64 view of the 2 CFL maxima words the next step reads (max-reduce them across strips)."""
        import torch
        ptr = C.c_void_p()
        self._check(self._L.swof_cfl_maxima(self._ctx, C.byref(ptr)))
        return self._view(ptr.value, 16, torch.int64)

    def cfl_maxima_addr(self) -> int:
        ptr = C.c_void_p()
        self._check(self._L.swof_cfl_maxima(self._ctx, C.byref(ptr)))
        return ptr.value

    def refresh_cfl(self):
        self._check(self._L.swof_refresh_cfl(self._ctx))

    def set_limits(self, t_end: float = float("inf"), step_limit: int = (1 << 63) - 1):
        self._check(self._L.swof_set_limits(self._ctx, float(t_end), int(step_limit)))

    def sync(self):
        self._check(self._L.swof_sync(self._ctx))

    def launches_per_step(self) -> int:
        """Kernel launches one time step of this context issues."""
        return self._L.swof_ctx_launches_per_step(self._ctx)


def selftest_math(n: int = 1 << 24, seed: int = 1307):
    """Bitwise mismatches (rcp, div, sqrt) of the kernels' IEEE operations vs CUDA's library ones."""
    out = (C.c_int64 * 3)()
    rc = lib().swof_selftest_math(int(n), int(seed), out)
    if rc != SWOF_OK:
        raise SwofError(rc, "selftest_math failed")
    return tuple(out)


def flow_direction(z, out=None, stream=None):
    """D8 flow direction (include/swof.h swof_flow_direction) of a (ny, nx) DEM: numpy or torch, host or
    CUDA, float64 or float32.  Returns `out` (uint8 codes 0..8; allocated like z if None)."""
    L = lib()
    is_torch = hasattr(z, "data_ptr")
    if is_torch:
        import torch
        assert z.is_contiguous() and z.dim() == 2 and z.dtype in (torch.float64, torch.float32)
        ny, nx = z.shape
        f32 = z.dtype == torch.float32
        if out is None:
            out = torch.empty((ny, nx), dtype=torch.uint8, device=z.device)
        zp = C.c_void_p(z.data_ptr())
        if stream is None and z.is_cuda:
            stream = torch.cuda.current_stream(z.device)
    else:
        z = np.ascontiguousarray(z)
        assert z.ndim == 2 and z.dtype in (np.float64, np.float32)
        ny, nx = z.shape
        f32 = z.dtype == np.float32
        if out is None:
            out = np.empty((ny, nx), dtype=np.uint8)
        zp = C.c_void_p(z.ctypes.data)
    op = C.c_void_p(out.data_ptr()) if hasattr(out, "data_ptr") else C.c_void_p(out.ctypes.data)
    sp = C.c_void_p(stream.cuda_stream) if stream is not None else None
    fn = L.swof_flow_direction_f32 if f32 else L.swof_flow_direction
    rc = fn(zp, nx, ny, op, sp)
    if rc != SWOF_OK:
        raise SwofError(rc, L.swof_strerror(rc).decode())
    return out


def ipc_open(handle: bytes) -> int:
    """Map a neighbour's workspace (swof_ipc_open); returns its base address in this process."""
    L = lib()
    p = C.c_void_p()
    buf = (C.c_ubyte * 64).from_buffer_copy(handle)
    rc = L.swof_ipc_open(buf, C.byref(p))
    if rc != SWOF_OK:
        raise SwofError(rc, "swof_ipc_open failed")
    return p.value


def ipc_close(base: int):
    lib().swof_ipc_close(C.c_void_p(base))


def copy(dst: int, src: int, nbytes: int, stream=None):
    """swof_copy: enqueue a copy between device addresses (ints) on `stream` (a torch.cuda.Stream)."""
    rc = lib().swof_copy(C.c_void_p(dst), C.c_void_p(src), nbytes, C.c_void_p(stream.cuda_stream) if stream else None)
    if rc != SWOF_OK:
        raise SwofError(rc, "swof_copy failed")
