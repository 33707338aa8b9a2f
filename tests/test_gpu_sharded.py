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


def sharded_run(cfg, nranks, nsteps, fused=False):
    import torch
    from paper_1307_4839_b200.sharded import LocalExchanger, ShardedSolver
    s = ShardedSolver(cfg, nranks, range(nranks), LocalExchanger(), stream=torch.cuda.Stream(), fused=fused)
    s.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf if cfg.ga is not None else None, 0.0)
    s.step(nsteps)
    out = s.get_state()
    out["dt"] = s.dt_history()
    s.close()
    return out


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("name,nx,ny,nranks,steps,kw", [
    ("cfg0", 64, 64, 2, 60, {}),
    ("cfg0", 64, 64, 3, 60, {}),
    ("cfg4", 75, 41, 3, 80, {}),
    ("cfg3", 130, 90, 4, 60, {}),          # W inflow segment cut by the strips, per-cell n, E free
    ("cfg1", 100, 70, 5, 60, {}),
    ("cfg4", 75, 41, 2, 40, {"cfl_mode": "face", "flux": "rusanov"}),
    ("cfg0", 64, 64, 2, 40, {"order": 1, "cfl": 1.0}),
])
def test_strips_equal_undivided(gpu, name, nx, ny, nranks, steps, kw, fused):
    """fused: the stage kernels store their boundary rows straight into the neighbours' ghost rows."""
    cfg = make(name, nx=nx, ny=ny)
    cfg.steps, cfg.t_end = steps, None
    for k, v in kw.items():
        setattr(cfg, k, v)
    whole = gpu_run(cfg, nsteps=steps)
    parts = sharded_run(cfg, nranks, steps, fused=fused)
    assert parts["step"] == whole["step"] == steps and parts["t"] == whole["t"]
    for k in ("h", "hu", "hv"):
        assert np.array_equal(parts[k], whole[k]), k
    if cfg.ga is not None:
        assert np.array_equal(parts["v"], whole["v"])
    assert np.array_equal(parts["dt"], whole["dt"])
    r = oracle.run(cfg)
    compare(parts, r, TOL_FULL)
    dt_close(parts["dt"], r["dt"])


def _ipc_worker(rank, world, port, name, nx, ny, steps, q):
    """One strip per process on the same GPU, neighbours' workspaces mapped with CUDA IPC, fused pushes,
    host barriers between phases (no kernel ever waits on another process's kernel)."""
    import os
    import torch
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_1307_4839_b200.sharded import IpcExchanger, ShardedSolver
        cfg = make(name, nx=nx, ny=ny)
        s = ShardedSolver(cfg, world, [rank], IpcExchanger(rank, world), stream=torch.cuda.Stream(), fused=True)
        s.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf if cfg.ga is not None else None, 0.0)
        s.step(steps)
        st = s.get_state()
        dt = s.dt_history()
        s.close()
        allst = [None] * world
        dist.all_gather_object(allst, (st, dt))
        dist.destroy_process_group()
        if rank == 0:
            q.put(("ok", allst))
        else:
            q.put(("ok", None))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put(("err", traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_ipc_fused_strips_two_processes(gpu, world):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    name, nx, ny, steps = "cfg4", 75, 41, 30
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, name, nx, ny, steps, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=120)
    errs = [r[1] for r in res if r[0] != "ok"]
    assert not errs, errs[0]
    allst = next(r[1] for r in res if r[1] is not None)
    cfg = make(name, nx=nx, ny=ny)
    cfg.steps, cfg.t_end = steps, None
    whole = gpu_run(cfg, nsteps=steps)
    for k in ("h", "hu", "hv", "v"):
        got = np.concatenate([st[k] for st, _ in allst], axis=0)
        assert np.array_equal(got, whole[k]), k
    assert np.array_equal(allst[0][1], whole["dt"])
