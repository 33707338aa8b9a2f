"""Pins of the oracle's D8 flow direction (user function listed at P:683-708;
SURVEY.md §8f NEXT(4)).  The neighbour enumeration E, SE, S, SW, W, NW, N, NE (codes 1..8, 0 = no
lower positive neighbour) and the examples are SPEC.md's `flow_direction`; rows (j) grow
northwards.  The brute-force check re-derives the defining property with numpy on random rasters.
"""
import numpy as np
import pytest

import oracle
from workloads.dem import NODATA, make_dem

# (di, dj) of codes 1..8: E, SE, S, SW, W, NW, N, NE (S = row j - 1)
OFFS = [(1, 0), (1, -1), (0, -1), (-1, -1), (-1, 0), (-1, 1), (0, 1), (1, 1)]


def test_spec_examples():
    assert np.all(oracle.flow_direction(np.full((5, 4), 7.0)) == 0)          # all equal -> 0
    # centre 5 with neighbours [9,9,9,9,1,9,9,9] in E, SE, S, SW, W, NW, N, NE order -> 5 (W)
    z = np.full((3, 3), 9.0)
    z[1, 1] = 5.0
    z[1, 0] = 1.0
    assert oracle.flow_direction(z)[1, 1] == 5


@pytest.mark.parametrize("code", range(1, 9))
def test_each_direction(code):
    di, dj = OFFS[code - 1]
    z = np.full((3, 3), 9.0)
    z[1, 1] = 5.0
    z[1 + dj, 1 + di] = 2.0
    assert oracle.flow_direction(z)[1, 1] == code
    assert oracle.flow_direction(z.astype(np.float32))[1, 1] == code


def test_ties_nodata_and_edges():
    z = np.full((3, 3), 9.0)
    z[1, 1] = 5.0
    z[0, 1] = 2.0          # S (code 3)
    z[2, 1] = 2.0          # N (code 7): equal, later in the order -> not taken (strict <)
    assert oracle.flow_direction(z)[1, 1] == 3
    z[1, 2] = NODATA       # E: lowest value but not > 0 -> skipped
    z[1, 0] = 0.0          # W: 0 is not > 0 either
    assert oracle.flow_direction(z)[1, 1] == 3
    # corner (0, 0) sees only E, N, NE; the lower cell beyond the edge does not exist
    z = np.array([[5.0, 6.0], [7.0, 4.0]])
    d = oracle.flow_direction(z)
    assert d[0, 0] == 8                    # NE (1, 1) = 4 < 5
    assert d[1, 1] == 0                    # the lowest cell: a pit
    assert d[0, 1] == 7                    # (1, 0): N neighbour (1, 1) = 4 beats W (0, 0) = 5
    # a no-data cell itself: nothing is below -9999, so 0
    z = np.full((3, 3), 3.0)
    z[1, 1] = NODATA
    assert oracle.flow_direction(z)[1, 1] == 0


def brute_force(z):
    """Independent restatement of the defining property: the first neighbour (in code order) whose value
    is the minimum over the in-grid neighbours that are > 0 and below the cell."""
    ny, nx = z.shape
    out = np.zeros((ny, nx), np.uint8)
    for j in range(ny):
        for i in range(nx):
            cand = []
            for k, (di, dj) in enumerate(OFFS):
                ii, jj = i + di, j + dj
                if 0 <= ii < nx and 0 <= jj < ny and z[jj, ii] > 0 and z[jj, ii] < z[j, i]:
                    cand.append((z[jj, ii], k + 1))
            if cand:
                m = min(v for v, _ in cand)
                out[j, i] = min(c for v, c in cand if v == m)
    return out


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_brute_force_random(seed):
    rs = np.random.default_rng(seed)
    z = np.round(rs.uniform(-2, 10, size=(23, 31)))     # many ties and non-positive cells
    assert np.array_equal(oracle.flow_direction(z), brute_force(z))
    assert np.array_equal(oracle.flow_direction(z.astype(np.float32)), brute_force(z))


def test_descent_invariants_on_dem():
    """Every non-zero code points to a strictly lower positive in-grid cell, so following the codes
    never cycles; f32 and f64 agree when the values are exact in both."""
    z = make_dem(120, 90, quantum=0.25)
    d = oracle.flow_direction(z)
    ny, nx = z.shape
    jj, ii = np.nonzero(d)
    k = d[jj, ii].astype(int) - 1
    di = np.array([o[0] for o in OFFS])[k]
    dj = np.array([o[1] for o in OFFS])[k]
    tgt = z[jj + dj, ii + di]
    assert np.all(tgt > 0) and np.all(tgt < z[jj, ii])
    assert np.all((ii + di >= 0) & (ii + di < nx) & (jj + dj >= 0) & (jj + dj < ny))
    assert np.array_equal(oracle.flow_direction(z.astype(np.float32)), d)
    assert np.array_equal(d, brute_force(z))
