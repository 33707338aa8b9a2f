"""The marching stage kernel's decomposition edges (csrc/swof_march.cuh): a warp owns 28
columns (lanes 2..29 of 32) and marches down a segment of rows whose height the library picks at create time
(SWOF_MARCH_H forces it).  Strip widths around 28, segment heights from 1 row up, grids narrower than a strip
or shorter than a segment, and every boundary type on the strip / segment ends: one and several steps against
the oracle, bit for bit (the evaluation contract of DESIGN.md §3)."""
import copy

import numpy as np
import pytest

import oracle
from swof_testlib import compare, gpu_run
from workloads import make
from workloads.configs import Inflow

pytestmark = pytest.mark.gpu

BCS = {
    "walls": {"W": "wall", "E": "wall", "S": "wall", "N": "wall"},
    "periodic_x": {"W": "periodic", "E": "periodic", "S": "free", "N": "wall"},
    "periodic_y": {"W": "free", "E": "wall", "S": "periodic", "N": "periodic"},
    "free": {"W": "free", "E": "free", "S": "free", "N": "free"},
}


def _case(name, nx, ny, bc=None):
    cfg = make(name, nx=nx, ny=ny)
    cfg.clamp_fail = 1.0          # tiny grids clamp (in the oracle as on the GPU); compared bit for bit below
    if bc is not None:
        cfg = copy.copy(cfg)
        cfg.bc = dict(BCS[bc])
        cfg.inflow = {}
    return cfg


@pytest.mark.parametrize("mh", [1, 2, 5, 16, 64])
@pytest.mark.parametrize("name,nx,ny,bc", [
    ("cfg4", 27, 9, None), ("cfg4", 28, 65, "periodic_x"), ("cfg4", 29, 17, "periodic_y"),
    ("cfg4", 57, 130, "free"), ("cfg3", 84, 70, None), ("cfg2", 30, 33, "walls"), ("cfg4", 3, 3, None),
    ("cfg4", 1, 40, "walls"), ("cfg4", 40, 1, "walls")])
def test_march_edges_bitwise(gpu, monkeypatch, mh, name, nx, ny, bc):
    monkeypatch.setenv("SWOF_MARCH_H", str(mh))
    cfg = _case(name, nx, ny, bc)
    g = gpu_run(cfg, nsteps=4)
    r = oracle.run(cfg, nsteps=4)
    res = compare(g, r, 1e-11)
    assert res["bitwise"], res
    assert np.array_equal(g["dt"], r["dt"])


@pytest.mark.parametrize("mh", [3, 64])
def test_march_inflow_on_segment_ends(gpu, monkeypatch, mh):
    """An inflow segment on the south side, cut by strip ends in x, and one on the west side spanning segment
    ends in y."""
    monkeypatch.setenv("SWOF_MARCH_H", str(mh))
    cfg = _case("cfg3", 90, 50)
    cfg.bc = {"W": "inflow", "E": "free", "S": "inflow", "N": "wall"}
    w = cfg.inflow["W"]
    cfg.inflow = {"W": Inflow(k0=5, k1=44, hydro_t=list(w.hydro_t), hydro_q=list(w.hydro_q)),
                  "S": Inflow(k0=20, k1=61, hydro_t=list(w.hydro_t), hydro_q=list(w.hydro_q))}
    g = gpu_run(cfg, nsteps=6)
    r = oracle.run(cfg, nsteps=6)
    res = compare(g, r, 1e-11)
    assert res["bitwise"], res


@pytest.mark.parametrize("mh", [8, 16])
@pytest.mark.parametrize("name,nx,ny,bc", [("cfg4", 57, 130, None), ("cfg3", 84, 70, None), ("cfg4", 29, 40, "periodic_y")])
def test_march_short_tail_segments(gpu, monkeypatch, mh, name, nx, ny, bc):
    """The last wave's shorter segments (SWOF_MARCH_TAIL=2 forces them on grids this small)."""
    monkeypatch.setenv("SWOF_MARCH_H", str(mh))
    monkeypatch.setenv("SWOF_MARCH_TAIL", "2")
    cfg = _case(name, nx, ny, bc)
    g = gpu_run(cfg, nsteps=4)
    r = oracle.run(cfg, nsteps=4)
    res = compare(g, r, 1e-11)
    assert res["bitwise"], res
