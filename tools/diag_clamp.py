"""Locate the first clamp > 1e-10 m on a full-size workload and check it against the oracle patch step.

    python tools/diag_clamp.py [cfg4] [max_steps]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import oracle  # noqa: E402
from swof_testlib import gpu_solver, oracle_patch_step  # noqa: E402
from workloads import make  # noqa: E402


def muscl_face_speeds(h, hu, hv, z, eps=1e-12, g=9.81):
    """max over x faces of |u_face| + sqrt(g h_face) (numpy, interior faces only) vs cell-centred bounds."""
    rh = np.where(h > eps, 1.0 / np.where(h > eps, h, 1.0), 0.0)
    u = hu * rh
    c = np.sqrt(g * h)
    return float(np.max(np.abs(u) + c)), float(np.max(np.abs(u)) + np.max(c))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    nmax = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    cfg = make(name)
    s = gpu_solver(cfg)
    prev = s.get_state()
    for k in range(nmax):
        try:
            s.step(1)
        except Exception as e:  # noqa: BLE001
            d = s.diag()
            print("step", k, "->", e, d)
            cell = d["big_clamp_cell"]
            j, i = divmod(cell, cfg.nx)
            print("clamp at cell", (i, j), "state before: h", prev["h"][j - 2:j + 3, i - 2:i + 3])
            dt = s.dt_history()[-1]
            sl, r, valid = oracle_patch_step(cfg, prev, prev["t"], dt, i, j)
            print("oracle patch counters:", r["counters"].as_dict())
            print("dt", dt, "t", prev["t"])
            print("cell-centred max(|u|+c) vs max|u| + max c:", muscl_face_speeds(prev["h"], prev["hu"], prev["hv"], cfg.z))
            jj, ii = slice(max(j - 3, 0), j + 4), slice(max(i - 3, 0), i + 4)
            np.set_printoptions(precision=4, linewidth=200)
            for key in ("h", "hu", "hv"):
                print(key, "\n", prev[key][jj, ii])
            print("z\n", cfg.z[jj, ii])
            return
        prev = s.get_state()
        d = s.diag()
        print("step", k, "t", d["t"], "dt", s.dt_history()[-1], "clamps", d["clamps"], "clamp_max", d["clamp_max"],
              flush=True)


if __name__ == "__main__":
    main()
