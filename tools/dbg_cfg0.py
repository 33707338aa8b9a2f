"""Locate cells where the GPU and the oracle differ bitwise (cfg0, a few steps)."""
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import oracle  # noqa: E402
from swof_testlib import gpu_run, gpu_solver  # noqa: E402
from workloads import make  # noqa: E402

for n in (1, 2, 3):
    cfg = make("cfg0", steps=n)
    g = gpu_run(cfg, nsteps=n)
    r = oracle.run(cfg)
    print("steps", n, "dt equal", np.array_equal(g["dt"], r["dt"]))
    for k in ("h", "hu", "hv"):
        d = np.nonzero(g[k] != r[k])
        print(" ", k, len(d[0]))
        for j, ii in list(zip(*d))[:4]:
            print("    ", j, ii, repr(g[k][j, ii]), repr(r[k][j, ii]), "h", repr(g["h"][j, ii]))
# one corrector stage from an identical U*
cfg = make("cfg0", steps=1)
P = oracle.params_from_config(cfg)
dt, _, _ = oracle.cfl_dt(P, cfg.h, cfg.hu, cfg.hv)
s = gpu_solver(cfg)
p = s.predictor()
r1 = oracle.stage(P, cfg.z, None, cfg.h, cfg.hu, cfg.hv, None, 0.0, dt)
r2 = oracle.stage(P, cfg.z, None, r1[0], r1[1], r1[2], None, dt, dt)
hn = 0.5 * (cfg.h + r2[0]); hun = 0.5 * (cfg.hu + r2[1])
s.step(1)
g = s.get_state()
d = np.nonzero(g["hu"] != hun)
print("manual heun hu diffs", len(d[0]), [(j, i, repr(g["hu"][j, i]), repr(hun[j, i]), repr(r2[1][j, i]), repr(cfg.hu[j, i])) for j, i in list(zip(*d))[:4]])
