"""C-ABI edge behaviour on the GPU (include/swof.h): swof_run's step cap saturates, and a clamp above
clamp_fail halts stepping at (or one step before) the failing step, the state then equal to the oracle's
after that many steps (SPEC's NegativeHeight abort; DESIGN.md §3 Q17)."""
import numpy as np
import pytest

import oracle
from swof_testlib import compare, gpu_solver
from workloads import make

pytestmark = pytest.mark.gpu

INT64_MAX = (1 << 63) - 1


def test_run_max_steps_saturates(gpu):
    """swof_step(1) then swof_run(t_end, INT64_MAX): 'no cap' must not wrap into 'no steps'."""
    cfg = make("cfg0", steps=10)
    s = gpu_solver(cfg)
    s.step(1)
    t1 = s.get_state()["t"]
    n = s.run(t1 + 1.0, INT64_MAX)
    g = s.get_state()
    s.close()
    assert n > 1 and g["t"] == t1 + 1.0 and g["step"] == 1 + n
    # the same through the oracle: step 1, then run to t1 + 1 s
    r1 = oracle.run(cfg, nsteps=1)
    r = oracle.run(cfg, h=r1["h"], hu=r1["hu"], hv=r1["hv"], t0=r1["t"], nsteps=1 << 40, t_end=t1 + 1.0)
    assert r["steps"] == n
    compare(g, r, 1e-11)


def test_bigclamp_halts_at_failing_step(gpu):
    """Rusanov at n_CFL 0.9 on a 96x64 cfg4 crop clamps 7.5 cm in its first step (its positivity needs a
    smaller CFL).  With clamp_fail = 1 mm the GPU stops at the step whose clamp exceeded it (the
    corrector's clamp completes that step, a predictor's aborts it) and the other 39 requested steps are
    no-ops; with clamp_fail = 1 m the same run takes all 40 steps."""
    from paper_1307_4839_b200 import SwofError
    fail = 1e-3
    cfg = make("cfg4", nx=96, ny=64, steps=40)
    cfg.flux, cfg.cfl, cfg.clamp_fail = "rusanov", 0.9, fail
    # the oracle's first step with a clamp above 1 mm (the oracle clamps and continues)
    k_fail = None
    for k in range(1, 41):
        r = oracle.run(cfg, nsteps=k)
        if r["counters"].clamp_max > fail:
            k_fail = k
            break
    assert k_fail is not None
    s = gpu_solver(cfg)
    with pytest.raises(SwofError) as ei:
        s.step(40)
    assert ei.value.code == 2                       # SWOF_ENUMERIC
    g = s.get_state()
    d = s.diag()
    s.close()
    assert d["flags"] & 2 and d["clamp_max"] > fail
    assert g["step"] in (k_fail - 1, k_fail), (g["step"], k_fail)
    r = oracle.run(cfg, nsteps=g["step"])
    compare(g, r, 1e-11)
    cfg.clamp_fail = 1.0
    s = gpu_solver(cfg)
    s.step(40)
    assert s.get_state()["step"] == 40 and s.diag()["flags"] == 0
    s.close()
