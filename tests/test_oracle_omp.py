"""The OpenMP-over-rows build of the oracle (liboracle_omp.so; used by tools/oracle_digests.py for the full-size
digests) gives the serial oracle's state bit for bit: each element is the same expression of the same inputs;
only the row loops are split over threads."""
import numpy as np
import pytest

import oracle
from workloads import make


@pytest.mark.parametrize("name,nx,ny,steps", [("cfg1", 160, 90, 40), ("cfg2", 97, 130, 30), ("cfg3", 140, 96, 40),
                                              ("cfg4", 211, 123, 15)])
def test_omp_build_bitwise(name, nx, ny, steps):
    cfg = make(name, nx=nx, ny=ny)
    cfg.steps, cfg.t_end = steps, None
    a = oracle.run(cfg)
    b = oracle.run(cfg, omp=True)
    assert a["steps"] == b["steps"] == steps and a["t"] == b["t"]
    for k in ("h", "hu", "hv", "dt"):
        assert np.array_equal(a[k], b[k]), k
    if cfg.ga is not None:
        assert np.array_equal(a["v"], b["v"])
    assert a["counters"].clamps == b["counters"].clamps and a["counters"].face_mid == b["counters"].face_mid
