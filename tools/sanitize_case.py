"""Small end-to-end run of every kernel for compute-sanitizer: cfg0 (walls) and a 256^2
cfg4 case through the graph path, a variant case (generic instance, order-1 commit, face CFL), the dry-row
skip, 2 row strips
(fused push), the D8 kernel (fp32 and fp64) and the math self-test."""
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1307_4839_b200 import Solver, flow_direction, params_from_config  # noqa: E402
from paper_1307_4839_b200.sharded import LocalExchanger, ShardedSolver  # noqa: E402
from paper_1307_4839_b200.swof import selftest_math  # noqa: E402
from workloads import make  # noqa: E402

torch.cuda.set_device(0)
for name, nx, ny, steps, kw in (("cfg0", None, None, 20, {}), ("cfg4", 256, 256, 20, {}),
                                ("cfg3", 130, 90, 10, {"flux": "rusanov", "order": 1, "cfl": 1.0, "cfl_mode": "face",
                                                       "ga_form": "darcy"}),
                                ("cfg3", 130, 90, 10, {"dry_skip": 1})):    # the dry-row skip instances
    cfg = make(name, nx=nx, ny=ny)
    for k, v in kw.items():
        setattr(cfg, k, v)
    s = Solver(params_from_config(cfg, graph_steps=8), cfg.z, cfg.fric_field)
    s.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf if cfg.ga is not None else None, 0.0)
    from paper_1307_4839_b200 import lib as _lib
    print("  after set_state", _lib().swof_check_line())
    s.step(steps)
    s.predictor()
    s.step_profiled(2)
    st = s.get_state()
    print(name, st["step"], s.diag()["volume"])
    s.close()
cfg = make("cfg4", nx=75, ny=41)
sh = ShardedSolver(cfg, 2, range(2), LocalExchanger(), fused=True)
sh.set_state(cfg.h, cfg.hu, cfg.hv, cfg.vinf, 0.0)
sh.step(5)
print("strips", sh.get_state()["step"])
sh.close()
z = np.round(np.random.default_rng(1).uniform(-2, 30, size=(70, 300)) * 2) / 2
print("d8", flow_direction(z).sum(), flow_direction(z.astype(np.float32)).sum())
print("math", selftest_math(1 << 16))
torch.cuda.synchronize()
from paper_1307_4839_b200 import lib  # noqa: E402
print("check_line", lib().swof_check_line())
print("done")
