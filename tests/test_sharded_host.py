"""Host logic of the row-strip decomposition (paper_1307_4839_b200/sharded.py): strip
partition and per-strip problem statements, and the torch.distributed halo exchange / CFL all-reduce at
world size 2 and 3 over gloo on CPU (mock strips with host tensors laid out like the library's fields:
2 ghost rows below and above)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1307_4839_b200.sharded import DistExchanger, LocalExchanger, strip_config, strip_rows
from workloads import make

SIDE_S, SIDE_N = 2, 3


def test_strip_rows_partition():
    for ny, n in ((41, 3), (64, 2), (90, 4), (8192, 8), (7, 3)):
        rows = [strip_rows(ny, n, r) for r in range(n)]
        assert rows[0][0] == 0 and rows[-1][1] == ny
        assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
        sizes = [b - a for a, b in rows]
        assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 2
    with pytest.raises(ValueError):
        strip_rows(5, 3, 0)


def test_strip_config_slices_and_sides():
    cfg = make("cfg3", nx=40, ny=90)          # W inflow segment rows 35..55, per-cell n, E free
    n = 4
    parts = [strip_config(cfg, r, n) for r in range(n)]
    assert parts[0].bc["S"] == cfg.bc["S"] and parts[0].bc["N"] == "halo"
    assert parts[-1].bc["N"] == cfg.bc["N"] and parts[-1].bc["S"] == "halo"
    assert all(p.bc["S"] == p.bc["N"] == "halo" for p in parts[1:-1])
    assert np.array_equal(np.concatenate([p.z for p in parts]), cfg.z)
    assert np.array_equal(np.concatenate([p.fric_field for p in parts]), cfg.fric_field)
    fl = cfg.inflow["W"]
    got = []
    for r, p in enumerate(parts):
        j0, _ = strip_rows(cfg.ny, n, r)
        if "W" in p.inflow:
            q = p.inflow["W"]
            assert q.width == (fl.k1 - fl.k0) * cfg.dy and q.hydro_q == fl.hydro_q
            got += list(range(j0 + q.k0, j0 + q.k1))
        else:
            assert p.bc["W"] == "wall"
    assert got == list(range(fl.k0, fl.k1))   # the segment is covered exactly once


class MockStrip:
    """Fields of a strip as the library lays them out: (ny + 4) x pitch, row 0 at offset 2 rows."""

    def __init__(self, rows, pitch, nsets=3, fill=0.0):
        self.rows, self.pitch = rows, pitch
        self.f = {s: [torch.full(((rows + 4) * pitch,), fill, dtype=torch.float64) for _ in range(3 if s < 2 else 1)]
                  for s in range(nsets)}
        self.words = torch.zeros(2, dtype=torch.int64)

    def halo_rows(self, s, side):
        b = 2 * self.pitch
        if side == SIDE_S:
            return [t[b:2 * b] for t in self.f[s]], [t[0:b] for t in self.f[s]]
        n = (self.rows + 2) * self.pitch
        return [t[n - b:n] for t in self.f[s]], [t[n:n + b] for t in self.f[s]]

    def cfl_maxima(self):
        return self.words


def fill_interior(st, rank, pitch):
    for s, ts in st.f.items():
        for k, t in enumerate(ts):
            v = t.view(st.rows + 4, pitch)
            for j in range(st.rows):
                v[j + 2] = 1000 * rank + 100 * s + 10 * k + j


def check_ghosts(st, rank, nranks, pitch, rows_of):
    for s, ts in st.f.items():
        for k, t in enumerate(ts):
            v = t.view(st.rows + 4, pitch)
            if rank > 0:       # S ghosts = the last 2 rows of the strip below
                rb = rows_of(rank - 1)
                assert torch.all(v[0] == 1000 * (rank - 1) + 100 * s + 10 * k + rb - 2)
                assert torch.all(v[1] == 1000 * (rank - 1) + 100 * s + 10 * k + rb - 1)
            if rank < nranks - 1:
                assert torch.all(v[st.rows + 2] == 1000 * (rank + 1) + 100 * s + 10 * k + 0)
                assert torch.all(v[st.rows + 3] == 1000 * (rank + 1) + 100 * s + 10 * k + 1)


def _worker(rank, world, port, ny, pitch, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        j0, j1 = strip_rows(ny, world, rank)
        st = MockStrip(j1 - j0, pitch)
        fill_interior(st, rank, pitch)
        ex = DistExchanger(rank, world)
        for s in (0, 1, 2):
            ex.exchange([st], s)
        check_ghosts(st, rank, world, pitch, lambda r: strip_rows(ny, world, r)[1] - strip_rows(ny, world, r)[0])
        st.words[:] = torch.tensor([rank * 7 + 3, 100 - rank], dtype=torch.int64)
        ex.allreduce_max([st.words])
        assert st.words.tolist() == [(world - 1) * 7 + 3, 100]
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_dist_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 23, 8, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: "ok" for r in range(world)}, res


def test_local_exchange_matches_dist_semantics():
    ny, n, pitch = 23, 3, 8
    strips = []
    for r in range(n):
        j0, j1 = strip_rows(ny, n, r)
        st = MockStrip(j1 - j0, pitch)
        fill_interior(st, r, pitch)
        strips.append(st)
    ex = LocalExchanger()
    for s in (0, 1, 2):
        ex.exchange(strips, s)
    for r, st in enumerate(strips):
        check_ghosts(st, r, n, pitch, lambda q: strip_rows(ny, n, q)[1] - strip_rows(ny, n, q)[0])
    for r, st in enumerate(strips):
        st.words[:] = torch.tensor([r, 10 - r], dtype=torch.int64)
    ex.allreduce_max([st.words for st in strips])
    assert all(st.words.tolist() == [n - 1, 10] for st in strips)
