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


def test_chunked_digest_run_equals_one_run(tmp_path):
    """tools/oracle_digests.py's resumable chunked run (used for the full-size digests that outlast one GPU-box
    call) gives the one-call run's state and dt sequence bit for bit, for a step-count and a t_end horizon."""
    import sys
    import time
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    import oracle_digests as od
    for name, kw, t_end in (("cfg3", dict(nx=90, ny=64, steps=70), None), ("cfg2", dict(nx=61, ny=47), 40.0)):
        cfg = make(name, **kw)
        if t_end is not None:
            cfg.t_end = t_end
        a = oracle.run(cfg, omp=True)
        r, _ = od.run_chunked(cfg, name, tmp_path, 0.0, time.time(), chunk=20)
        assert r is None                              # checkpointed after the first chunk
        while r is None:
            r, _ = od.run_chunked(cfg, name, tmp_path, 0.0, time.time(), chunk=20)
        for k in ("h", "hu", "hv", "dt"):
            assert np.array_equal(a[k], r[k]), (name, k)
        assert a["t"] == r["t"] and a["steps"] == r["steps"]
