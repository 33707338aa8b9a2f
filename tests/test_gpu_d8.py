"""T4 for the D8 flow direction: the sm_100a kernel through the C ABI against the
oracle (listing P:683-708), bit-exact (integer codes), fp64 and fp32 rasters, host
and device pointers, ragged and degenerate sizes, ties and no-data, and the paper's 14786 x 10086 size.
"""
import numpy as np
import pytest

import oracle
from workloads.dem import DEM_SIZES, make_dem

pytestmark = pytest.mark.gpu


def rand_raster(nx, ny, seed):
    rs = np.random.default_rng(seed)
    z = np.round(rs.uniform(-3.0, 40.0, size=(ny, nx)) * 4.0) / 4.0     # ties and non-positive values
    return np.ascontiguousarray(z)


@pytest.mark.parametrize("nx,ny", [(1, 1), (1, 300), (300, 1), (2, 2), (129, 17), (130, 18), (257, 33),
                                   DEM_SIZES["dem_small"]])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_d8_parity_host(gpu, nx, ny, dtype):
    from paper_1307_4839_b200 import flow_direction
    z = rand_raster(nx, ny, nx * 7 + ny).astype(dtype)
    assert np.array_equal(flow_direction(z), oracle.flow_direction(z))


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_d8_parity_device_pointers(gpu, dtype):
    import torch
    from paper_1307_4839_b200 import flow_direction
    z = make_dem(*DEM_SIZES["dem_small"]).astype(dtype)
    zt = torch.from_numpy(z).cuda()
    out = flow_direction(zt)
    torch.cuda.synchronize()
    assert out.is_cuda and out.dtype == torch.uint8
    assert np.array_equal(out.cpu().numpy(), oracle.flow_direction(z))


def test_d8_paper_size(gpu):
    """The paper's large DEM size, whole raster compared, both precisions."""
    import torch
    from paper_1307_4839_b200 import flow_direction
    nx, ny = DEM_SIZES["dem_large"]
    z = make_dem(nx, ny)
    for zz in (z, z.astype(np.float32)):
        ref = oracle.flow_direction(zz)
        got = flow_direction(torch.from_numpy(zz).cuda()).cpu().numpy()
        assert np.array_equal(got, ref)
        counts = np.bincount(got.ravel(), minlength=9)
        assert counts.sum() == nx * ny and counts[1:].min() > 0


def test_d8_rejects_bad_arguments(gpu):
    import ctypes as C
    from paper_1307_4839_b200 import lib
    L = lib()
    buf = np.zeros((4, 4))
    out = np.zeros((4, 4), np.uint8)
    assert L.swof_flow_direction(None, 4, 4, C.c_void_p(out.ctypes.data), None) == 1
    assert L.swof_flow_direction(C.c_void_p(buf.ctypes.data), 0, 4, C.c_void_p(out.ctypes.data), None) == 1
