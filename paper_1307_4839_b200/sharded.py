"""Row-strip domain decomposition of the time step (the paper's MPI design,
P:731-760: "the domain is cut into sub-domains ... exchanging the points on the interfaces").

Host orchestration only -- argument marshalling and collective plumbing; every arithmetic step runs in
the CUDA kernels of libswof.so.  The grid's rows are split into balanced strips, one per rank (one GPU
per process over NCCL/NVLink with torch.distributed), or several strips driven from one process (the
LocalExchanger: used to check the decomposition on a single device).  A strip is an ordinary context
whose S/N sides are SWOF_BC_HALO; each time step is

    phase 0 (predictor) -> halo exchange of U* -> phase 1 (corrector) -> halo exchange of U^{n+1}
    -> phase 2 (face CFL, if any) -> all-reduce(max) of the 2 CFL words

so that every strip computes exactly what the undivided grid computes on its rows (bit for bit).
"""
from __future__ import annotations

import copy

import numpy as np

from .swof import SIDE_N, SIDE_S, Solver, copy as dev_copy, ipc_close, ipc_open, params_from_config


def strip_rows(ny: int, nranks: int, rank: int):
    """Rows [j0, j1) of strip `rank`: balanced, the first ny % nranks strips one row longer."""
    if not 0 <= rank < nranks or ny < 2 * nranks:
        raise ValueError(f"cannot cut {ny} rows into {nranks} strips of >= 2 rows")
    base, extra = divmod(ny, nranks)
    j0 = rank * base + min(rank, extra)
    return j0, j0 + base + (1 if rank < extra else 0)


def strip_config(cfg, rank: int, nranks: int):
    """The problem statement of strip `rank`: its rows of every input, HALO on the cut sides, W/E inflow
    segments clipped to the strip with the global segment width (so q = Q/W is unchanged)."""
    if nranks > 1 and "periodic" in (cfg.bc["S"], cfg.bc["N"]):
        raise ValueError("periodic S/N boundaries are not supported by the strip decomposition")
    j0, j1 = strip_rows(cfg.ny, nranks, rank)
    s = copy.copy(cfg)
    s.ny = j1 - j0
    s.bc = dict(cfg.bc)
    if rank > 0:
        s.bc["S"] = "halo"
    if rank < nranks - 1:
        s.bc["N"] = "halo"
    s.inflow = {}
    for side, fl in cfg.inflow.items():
        if side in ("S", "N"):
            if s.bc[side] != "halo":
                s.inflow[side] = fl
            continue
        k0, k1 = max(fl.k0 - j0, 0), min(fl.k1 - j0, s.ny)
        if k0 >= k1:
            s.bc[side] = "wall"          # outside the segment an inflow side is a wall (Q18)
            continue
        w = fl.width if fl.width else (fl.k1 - fl.k0) * cfg.dy
        s.inflow[side] = type(fl)(k0=k0, k1=k1, hydro_t=list(fl.hydro_t), hydro_q=list(fl.hydro_q), width=w)
    for k in ("z", "h", "hu", "hv", "vinf", "fric_field"):
        a = getattr(cfg, k)
        setattr(s, k, None if a is None else np.ascontiguousarray(a[j0:j1]))
    return s


class LocalExchanger:
    """All strips in this process (one stream): halo rows are device-to-device copies, the CFL all-reduce
    a max over the strips' words.  Fused mode: the kernels push their boundary rows into the neighbours'
    ghost rows themselves (swof_set_halo_push) and stream order is the barrier."""

    def link_push(self, strips):
        for lo, hi in zip(strips[:-1], strips[1:]):
            lo.set_halo_push(SIDE_N, hi.halo_block_addrs(0, SIDE_S)[1], hi.halo_block_addrs(1, SIDE_S)[1])
            hi.set_halo_push(SIDE_S, lo.halo_block_addrs(0, SIDE_N)[1], lo.halo_block_addrs(1, SIDE_N)[1])

    def barrier(self, strips):
        pass

    def exchange(self, strips, field_set: int):
        for lo, hi in zip(strips[:-1], strips[1:]):
            lo_send, lo_recv = lo.halo_rows(field_set, SIDE_N)
            hi_send, hi_recv = hi.halo_rows(field_set, SIDE_S)
            for a, b in zip(lo_recv, hi_send):
                a.copy_(b)
            for a, b in zip(hi_recv, lo_send):
                a.copy_(b)

    def allreduce_max_strips(self, strips):
        self.allreduce_max([sv.cfl_maxima() for sv in strips])

    def allreduce_max(self, words):
        import torch
        m = words[0].clone()
        for w in words[1:]:
            m = torch.maximum(m, w)
        for w in words:
            w.copy_(m)


class DistExchanger:
    """One strip per rank over torch.distributed (NCCL on GPUs; gloo works for host tensors): send/recv of
    the 2-row blocks with the ranks below and above, all-reduce(max) of the CFL words (int64 view of
    non-negative IEEE doubles: integer order = value order)."""

    def __init__(self, rank: int, nranks: int, group=None):
        self.rank, self.nranks, self.group = rank, nranks, group

    def exchange(self, strips, field_set: int):
        import torch.distributed as dist
        (sv,) = strips
        ops = []
        if self.rank > 0:
            send, recv = sv.halo_rows(field_set, SIDE_S)
            ops += [dist.P2POp(dist.isend, t, self.rank - 1, self.group) for t in send]
            ops += [dist.P2POp(dist.irecv, t, self.rank - 1, self.group) for t in recv]
        if self.rank < self.nranks - 1:
            send, recv = sv.halo_rows(field_set, SIDE_N)
            ops += [dist.P2POp(dist.isend, t, self.rank + 1, self.group) for t in send]
            ops += [dist.P2POp(dist.irecv, t, self.rank + 1, self.group) for t in recv]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()

    def allreduce_max_strips(self, strips):
        self.allreduce_max([sv.cfl_maxima() for sv in strips])

    def allreduce_max(self, words):
        import torch.distributed as dist
        (w,) = words
        if self.nranks > 1:
            dist.all_reduce(w, op=dist.ReduceOp.MAX, group=self.group)


class IpcExchanger:
    """One strip per process, the neighbours' workspaces mapped with CUDA IPC (NVLink peer memory across
    GPUs; also valid between processes sharing one GPU).  Fused mode only: the kernels push boundary rows
    into the mapped neighbours; the state loaded by set_state is pulled once by copies.  Ordering between
    strips after each phase is either a host barrier (any backend: stream synchronise + dist.barrier; the
    mode the tests run, 2-3 processes sharing one GPU over gloo) or, with in_stream=True on an NCCL group,
    a one-word all-reduce enqueued on the strip's stream (no host round trip: the neighbours' producing
    kernels precede their all-reduce in stream order, so its completion orders their peer stores before
    this strip's next phase); the CFL all-reduce follows the same choice."""

    def __init__(self, rank: int, nranks: int, group=None, in_stream: bool = False):
        self.rank, self.nranks, self.group, self.in_stream = rank, nranks, group, in_stream
        self.peers = {}                       # side -> (mapped base, info dict of the neighbour)
        self._word = None                     # device scratch of the in-stream barrier / CFL all-reduce

    def _neighbours(self):
        out = {}
        if self.rank > 0:
            out[SIDE_S] = self.rank - 1
        if self.rank < self.nranks - 1:
            out[SIDE_N] = self.rank + 1
        return out

    def link_push(self, strips):
        import torch.distributed as dist
        (sv,) = strips
        if self.nranks == 1:
            return
        handle, base = sv.ipc_handle()
        info = {"handle": handle, "base": base, "blocks": {}}
        for side in (SIDE_S, SIDE_N):
            for fs in (0, 1, 2):
                send, recv, nb = sv.halo_block_addrs(fs, side)
                info["blocks"][(fs, side)] = ([a - base if a else 0 for a in send], [a - base if a else 0 for a in recv], nb)
        allinfo = [None] * self.nranks
        dist.all_gather_object(allinfo, info, group=self.group)
        opposite = {SIDE_S: SIDE_N, SIDE_N: SIDE_S}
        for side, nbr in self._neighbours().items():
            other = allinfo[nbr]
            mbase = ipc_open(other["handle"])
            self.peers[side] = (mbase, other)
            recv = [[mbase + off for off in other["blocks"][(fs, opposite[side])][1]] for fs in (0, 1)]
            sv.set_halo_push(side, recv[0], recv[1])
        self.barrier(strips)

    def exchange(self, strips, field_set: int):
        """Pull the neighbours' boundary rows of `field_set` into this strip's ghost rows (after a barrier)."""
        (sv,) = strips
        self.barrier(strips)
        opposite = {SIDE_S: SIDE_N, SIDE_N: SIDE_S}
        for side, (mbase, other) in self.peers.items():
            _, recv, nb = sv.halo_block_addrs(field_set, side)
            send_off, _, _ = other["blocks"][(field_set, opposite[side])]
            for dst, off in zip(recv, send_off):
                if dst and off:
                    dev_copy(dst, mbase + off, nb, sv.stream)
        self.barrier(strips)

    def _scratch(self, sv):
        import torch
        if self._word is None:
            self._word = torch.zeros(3, dtype=torch.int64, device=torch.cuda.current_device())
        return self._word

    def barrier(self, strips):
        import torch
        import torch.distributed as dist
        if self.nranks == 1:
            return
        if self.in_stream:
            (sv,) = strips
            w = self._scratch(sv)
            with torch.cuda.stream(sv.stream):
                dist.all_reduce(w[2:3], op=dist.ReduceOp.MAX, group=self.group)
            return
        for sv in strips:
            sv.stream.synchronize()
        dist.barrier(group=self.group)

    def allreduce_max_strips(self, strips):
        import torch
        import torch.distributed as dist
        (sv,) = strips
        if self.nranks == 1:
            return
        addr = sv.cfl_maxima_addr()
        if self.in_stream:
            w = self._scratch(sv)
            with torch.cuda.stream(sv.stream):
                dev_copy(w.data_ptr(), addr, 16, sv.stream)
                dist.all_reduce(w[0:2], op=dist.ReduceOp.MAX, group=self.group)
                dev_copy(addr, w.data_ptr(), 16, sv.stream)
            return
        host = torch.zeros(2, dtype=torch.int64)
        dev_copy(host.data_ptr(), addr, 16, sv.stream)
        sv.stream.synchronize()
        dist.all_reduce(host, op=dist.ReduceOp.MAX, group=self.group)
        dev_copy(addr, host.data_ptr(), 16, sv.stream)
        sv.stream.synchronize()

    def close(self):
        for mbase, _ in self.peers.values():
            ipc_close(mbase)
        self.peers = {}


class ShardedSolver:
    """The time step of `cfg` on row strips.  `ranks`: the strips this process drives (all of them with a
    LocalExchanger; its own rank with a DistExchanger)."""

    def __init__(self, cfg, nranks: int, ranks, exchanger, stream=None, graph_steps: int = 0, fused: bool = False):
        """fused: the stage kernels push their boundary rows into the neighbours' ghost rows themselves
        (no exchange pass; a barrier between phases); needs LocalExchanger or IpcExchanger."""
        import torch
        self.cfg, self.nranks, self.ranks, self.ex, self.fused = cfg, nranks, list(ranks), exchanger, fused
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        self.parts = [strip_config(cfg, r, nranks) for r in self.ranks]
        ipc = isinstance(exchanger, IpcExchanger)
        self.strips = [Solver(params_from_config(p, graph_steps=graph_steps), p.z, p.fric_field, stream=self.stream,
                              use_torch_workspace=not ipc) for p in self.parts]
        if fused or ipc:
            self.ex.link_push(self.strips)
        with torch.cuda.stream(self.stream):
            self.ex.exchange(self.strips, 2)                 # z ghost rows, once

    def set_state(self, h, hu, hv, v_inf=None, t0: float = 0.0):
        """Global (ny, nx) arrays; each strip takes its rows."""
        import torch
        for r, sv in zip(self.ranks, self.strips):
            j0, j1 = strip_rows(self.cfg.ny, self.nranks, r)
            sl = slice(j0, j1)
            sv.set_state(np.ascontiguousarray(h[sl]), np.ascontiguousarray(hu[sl]), np.ascontiguousarray(hv[sl]),
                         None if v_inf is None else np.ascontiguousarray(v_inf[sl]), t0)
        with torch.cuda.stream(self.stream):
            self.ex.exchange(self.strips, 0)
            for sv in self.strips:
                sv.refresh_cfl()
            self.ex.allreduce_max_strips(self.strips)
        for sv in self.strips:
            sv.sync()

    def step(self, nsteps: int, t_end: float = float("inf")):
        import torch
        for sv in self.strips:
            sv.set_limits(t_end)
        with torch.cuda.stream(self.stream):
            for _ in range(nsteps):
                for sv in self.strips:
                    sv.enqueue_phase(0)
                if self.fused:
                    self.ex.barrier(self.strips)             # U* rows already pushed by the predictor
                else:
                    self.ex.exchange(self.strips, 1)
                for sv in self.strips:
                    sv.enqueue_phase(1)
                if self.fused:
                    self.ex.barrier(self.strips)
                else:
                    self.ex.exchange(self.strips, 0)
                for sv in self.strips:
                    sv.enqueue_phase(2)
                self.ex.allreduce_max_strips(self.strips)
        for sv in self.strips:
            sv.sync()

    def get_state(self):
        """The driven strips' rows stacked (the whole grid with a LocalExchanger)."""
        outs = [sv.get_state() for sv in self.strips]
        res = {k: np.concatenate([o[k] for o in outs], axis=0) for k in ("h", "hu", "hv")}
        if outs[0].get("v") is not None:
            res["v"] = np.concatenate([o["v"] for o in outs], axis=0)
        res["t"], res["step"] = outs[0]["t"], outs[0]["step"]
        return res

    def dt_history(self):
        return self.strips[0].dt_history()

    def close(self):
        if hasattr(self.ex, "close"):
            self.ex.close()
        for sv in self.strips:
            sv.close()
