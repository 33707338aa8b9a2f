"""Row-strip decomposition on the GPU: all strips driven from one process on
one device with the LocalExchanger (the decomposition's data flow without needing several GPUs; the
multi-rank exchange itself is covered by tests/test_sharded_host.py over gloo).  The strips must
reproduce the undivided GPU run bit for bit -- same arithmetic, ghost rows carry the neighbours' values --
and the oracle within the parity tolerances."""
import numpy as np
import pytest

import oracle
from swof_testlib import compare, gpu_run
from test_gpu_parity import TOL_FULL, dt_close
from workloads import make

pytestmark = pytest.mark.gpu


def sharded_run(cfg, nranks, nsteps):
    import torch
    from paper_1307_4839_b200.sharded import LocalExchanger, ShardedSolver
    s = ShardedSolver(cfg, nranks, range(nranks), LocalExchanger(), stream=torch.cuda.Stream())
    s.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf if cfg.ga is not None else None, 0.0)
    s.step(nsteps)
    out = s.get_state()
    out["dt"] = s.dt_history()
    s.close()
    return out


@pytest.mark.parametrize("name,nx,ny,nranks,steps,kw", [
    ("cfg0", 64, 64, 2, 60, {}),
    ("cfg0", 64, 64, 3, 60, {}),
    ("cfg4", 75, 41, 3, 80, {}),
    ("cfg3", 130, 90, 4, 60, {}),          # W inflow segment cut by the strips, per-cell n, E free
    ("cfg1", 100, 70, 5, 60, {}),
    ("cfg4", 75, 41, 2, 40, {"cfl_mode": "face", "flux": "rusanov"}),
    ("cfg0", 64, 64, 2, 40, {"order": 1, "cfl": 1.0}),
])
def test_strips_equal_undivided(gpu, name, nx, ny, nranks, steps, kw):
    cfg = make(name, nx=nx, ny=ny)
    cfg.steps, cfg.t_end = steps, None
    for k, v in kw.items():
        setattr(cfg, k, v)
    whole = gpu_run(cfg, nsteps=steps)
    parts = sharded_run(cfg, nranks, steps)
    assert parts["step"] == whole["step"] == steps and parts["t"] == whole["t"]
    for k in ("h", "hu", "hv"):
        assert np.array_equal(parts[k], whole[k]), k
    if cfg.ga is not None:
        assert np.array_equal(parts["v"], whole["v"])
    assert np.array_equal(parts["dt"], whole["dt"])
    r = oracle.run(cfg)
    compare(parts, r, TOL_FULL)
    dt_close(parts["dt"], r["dt"])
