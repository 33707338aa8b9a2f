"""Maximum-size edge case: a grid of more than 2^31 cells (every flat cell index, every row offset and every
field's byte offset past 2^31) advanced through the C ABI, compared element by element with the oracle.

The oracle cannot step 2.15e9 cells, so the comparison uses a property that holds at any size (domain of
dependence, Algorithm 1 P:773-788 with the 2-cell stencil of MUSCL + HLL): the grid is a flat bed
under uniform rain with walls on all four sides, still water everywhere except a dam-break column on
a ramp in the north-east corner -- the cells at the highest addresses.  A still, uniform state stays
uniform and still exactly (equal states give equal face fluxes, their difference is 0; the wall mirror of a
uniform still state is that state), so after K steps every cell more than 4K cells away from the column is
the still rain state, and the CFL maxima are the column's.  The NE corner block of the grid is
therefore the same problem as that block on its own with walls on its cut sides: the oracle runs the block
(its cut-side ghosts are the still rain state too) and the GPU's corner must equal it cell for cell, with the
same dt sequence, bit for bit.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
from workloads.configs import SwofConfig, mm_per_h

pytestmark = pytest.mark.gpu

NX, NY = 46336, 46400          # 2 150 000 000+ cells; nx not a multiple of the 28 own columns of a strip
CY, CX = 200, 230              # the compared NE corner block (ragged against 32 / 28 / segment heights)
COL = 48                       # dam-break column in the corner, on a ramp
K = 20                         # steps: the disturbance reaches <= 4K = 80 cells from the column


def _problem(nx, ny):
    return SwofConfig(name="maxsize", nx=nx, ny=ny, dx=1.0, dy=1.0, cfl=0.4, dt_max=1.0, h_eps=1e-12,
                      fric_law="manning", fric_coef=0.03, rain_t=[0.0], rain_rate=[mm_per_h(50.0)],
                      bc={s: "wall" for s in ("W", "E", "S", "N")}, steps=K)


def _corner_fields(cy, cx):
    """h and z of the corner block (rows ny-cy.., cols nx-cx..): column of 1.2 m on a ramp, dry elsewhere."""
    h = np.zeros((cy, cx))
    z = np.zeros((cy, cx))
    jj, ii = np.meshgrid(np.arange(COL), np.arange(COL), indexing="ij")
    z[cy - COL:, cx - COL:] = 0.01 * (ii + 0.5 * jj)             # rises towards the NE walls
    h[cy - COL:, cx - COL:] = 1.2 - 0.5 * z[cy - COL:, cx - COL:]
    return h, z


def test_more_than_2_31_cells_corner_equals_oracle(gpu):
    import torch
    from paper_1307_4839_b200 import Solver, params_from_config
    from paper_1307_4839_b200.swof import _ptr, lib

    assert NX * NY > 2 ** 31 and (NY - 1) * NX > 2 ** 31
    cfg = _problem(NX, NY)
    P = params_from_config(cfg, graph_steps=4)
    L = lib()
    need = C.c_size_t()
    assert L.swof_workspace_size(C.byref(P), C.byref(need)) == 0
    free, _ = torch.cuda.mem_get_info()
    field = NY * NX * 8
    if free < need.value + field + (2 << 30):
        pytest.skip(f"needs {(need.value + field) / 1e9:.0f} GB of device memory, {free / 1e9:.0f} GB free")

    hc, zc = _corner_fields(CY, CX)
    # full-size host inputs: calloc'd zero pages (never touched) except the corner block
    z = np.zeros((NY, NX))
    h = np.zeros((NY, NX))
    zero = np.zeros((NY, NX))
    z[NY - CY:, NX - CX:] = zc
    h[NY - CY:, NX - CX:] = hc
    s = Solver(P, z, None)
    s.set_state(h, zero, zero, None, 0.0)
    del z, h, zero
    s.step(K)
    corner = {}
    out = torch.empty((NY, NX), dtype=torch.float64, device=s.device)
    for k, idx in (("h", 0), ("hu", 1), ("hv", 2)):
        ptrs = [None, None, None]
        ptrs[idx] = _ptr(out, s.shape)
        t, st = C.c_double(), C.c_int64()
        assert s._L.swof_get_state(s._ctx, *ptrs, None, C.byref(t), C.byref(st)) == 0
        torch.cuda.synchronize()
        corner[k] = out[NY - CY:, NX - CX:].cpu().numpy().copy()
        # far from the column: the still rain state, uniform over the whole grid (sampled rows, incl. row 0)
        far = out[:: NY // 7, : NX - CX - 100 : 997].cpu().numpy()
        assert np.all(far == far[0, 0]), k
    assert st.value == K
    dt_gpu = s.dt_history()
    diag = s.diag()
    del out
    s.close()
    torch.cuda.empty_cache()

    blk = _problem(CX, CY)
    blk.z = zc
    blk.h, blk.hu, blk.hv = hc, np.zeros((CY, CX)), np.zeros((CY, CX))
    r = oracle.run(blk, nsteps=K)
    assert r["steps"] == K
    assert np.array_equal(np.asarray(dt_gpu).view(np.int64), np.asarray(r["dt"])[:K].view(np.int64))
    for k in ("h", "hu", "hv"):
        g, o = corner[k], r[k]
        assert np.array_equal(g, o), (k, float(np.max(np.abs(g - o))))
        nz = (g != 0) | (o != 0)
        assert np.array_equal(g[nz].view(np.int64), o[nz].view(np.int64)), k   # bit for bit where nonzero
    # the disturbance stayed inside the block (the premise of the comparison)
    still = r["h"][: CY - COL - 4 * K - 8, : CX - COL - 4 * K - 8]
    assert np.all(still == still[0, 0]) and still[0, 0] > 0
    print(f"max-size: {NX}x{NY} = {NX * NY} cells, corner {CY}x{CX} bit-identical over {K} steps, "
          f"dt[-1] = {dt_gpu[-1]!r}, diag volume {diag['volume']:.6e}")
