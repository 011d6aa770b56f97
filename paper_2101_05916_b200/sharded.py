"""Multi-GPU slab-partitioned solve (one process per GPU).

Axis 0 of a 4D grid is split into balanced slabs (``slab_partition``, the
library's own rule); each rank solves its slab with NCCL halo exchange and a
residual all-reduce inside the device loop (``hjb_solve_sharded_dev``).
torch.distributed is only the plumbing that ships the NCCL unique id from
rank 0 to the others.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import abi
from . import hjsafe as hj


def slab_partition(n0: int, nranks: int, rank: int) -> tuple[int, int]:
    """Owned planes [begin, end) of `rank` (first n0 % nranks ranks get one more)."""
    b, e = C.c_int64(), C.c_int64()
    hj._check(abi.load().hjb_slab_partition(n0, nranks, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def sweep_planes_dev(grid: hj.Grid, model: hj.DynamicsModel, dbounds: hj.IntervalField,
                     value_ptr: int, c_ptr: int, plane_begin: int, plane_end: int, dt: float,
                     out_ptr: int, ctx: hj.Context | None = None) -> float:
    """One sweep of planes [plane_begin, plane_end) on a full grid (device
    pointers); returns the slab's max|dV|."""
    lib = abi.load()
    mx = C.c_double()
    g, m, d = grid.to_c(), model.to_c(), dbounds.to_c()
    hj._check(lib.hjb_sweep_planes_dev(hj._ctx(ctx), C.byref(g), C.byref(m), C.byref(d),
                                       C.c_void_p(value_ptr), C.c_void_p(c_ptr), plane_begin,
                                       plane_end, dt, C.c_void_p(out_ptr), C.byref(mx)))
    return mx.value


def ho_stage_planes_dev(grid: hj.Grid, model: hj.DynamicsModel, dbounds: hj.IntervalField,
                        stage_in_ptr: int, value_n_ptr: int, c_ptr: int, dt: float, order: int,
                        kind: int, plane_begin: int, plane_end: int, out_ptr: int,
                        ctx: hj.Context | None = None) -> float:
    """One ENO/TVD-RK stage of planes [plane_begin, plane_end) on a full grid
    (device pointers); returns the slab's max|out - V_n|."""
    lib = abi.load()
    mx = C.c_double()
    g, m, d = grid.to_c(), model.to_c(), dbounds.to_c()
    hj._check(lib.hjb_ho_stage_planes_dev(hj._ctx(ctx), C.byref(g), C.byref(m), C.byref(d),
                                          C.c_void_p(stage_in_ptr), C.c_void_p(value_n_ptr),
                                          C.c_void_p(c_ptr), dt, order, kind, plane_begin,
                                          plane_end, C.c_void_p(out_ptr), C.byref(mx)))
    return mx.value


def slab_plan(n0: int, nranks: int, rank: int, halo: int) -> dict:
    """The per-rank plan of the sharded solve (hjb_slab_plan, host only):
    local geometry, halo send/receive planes and the boundary/interior
    split, in the rank's local plane numbers."""
    out = (C.c_int64 * 16)()
    hj._check(abi.load().hjb_slab_plan(n0, nranks, rank, halo, out))
    keys = ["owned", "nloc", "cbeg", "cend", "global_begin", "send_lo", "recv_lo", "send_hi",
            "recv_hi", "halo", "b0", "e0", "b1", "e1", "i0", "i1"]
    return dict(zip(keys, list(out)))


class Comm:
    """Communicator of the library, bootstrapped over torch.distributed.

    p2p=False: NCCL (the unique id is broadcast by torch.distributed).
    p2p=True: the peer-store communicator, no NCCL: the ranks' control blocks
    are mapped over CUDA IPC (handles all-gathered by torch.distributed, any
    backend, e.g. gloo); every per-sweep exchange runs on the devices."""

    def __init__(self, ctx: hj.Context, rank: int, world: int, device, p2p: bool = False):
        import torch
        import torch.distributed as dist
        lib = abi.load()
        self.rank, self.world = rank, world
        if p2p:
            h = C.c_void_p()
            hj._check(lib.hjb_p2p_comm_create(ctx.handle, world, rank, C.byref(h)))
            self.handle = h
            mine = (C.c_uint8 * 64)()
            hj._check(lib.hjb_comm_ctl_handle(h, mine))
            allh = [bytes(mine)]
            if world > 1:
                allh = [None] * world
                dist.all_gather_object(allh, bytes(mine))
            buf = (C.c_uint8 * (64 * world)).from_buffer_copy(b"".join(allh))
            hj._check(lib.hjb_comm_open_peers(h, buf))
            return
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            hj._check(lib.hjb_nccl_unique_id(uid))
        t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=device)
        if world > 1:
            dist.broadcast(t, src=0)
        raw = bytes(t.cpu().tolist())
        buf = (C.c_uint8 * 128).from_buffer_copy(raw)
        h = C.c_void_p()
        hj._check(lib.hjb_comm_create(ctx.handle, world, rank, buf, C.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            abi.load().hjb_comm_destroy(self.handle)
            self.handle = None


def solve_sharded_dev(comm: Comm, grid: hj.Grid, model: hj.DynamicsModel,
                      dbounds: hj.IntervalField, init_ptr: int, c_ptr: int, out_ptr: int,
                      cfg: hj.SolveConfig, ctx: hj.Context, history_capacity: int = 0):
    """hjb_solve_sharded_dev: pointers hold this rank's owned planes."""
    lib = abi.load()
    r, rh, wh = hj._c_result(int(history_capacity))
    g, m, d, c = grid.to_c(), model.to_c(), dbounds.to_c(), cfg.to_c()
    hj._check(lib.hjb_solve_sharded_dev(ctx.handle, comm.handle, C.byref(g), C.byref(m), C.byref(d),
                                        C.c_void_p(init_ptr), C.c_void_p(c_ptr), C.byref(c),
                                        C.c_void_p(out_ptr), C.byref(r)))
    n = min(int(r.iterations), int(r.history_capacity))
    return hj.SolveResult(value=None, iterations=int(r.iterations), dt=float(r.dt),
                          wall_seconds=float(r.wall_seconds), converged=bool(r.converged),
                          residual_history=rh[:n].copy(), wall_ms_history=wh[:n].copy(),
                          nodes_per_sweep=int(r.nodes_per_sweep),
                          final_residual=float(r.final_residual))


def solve_sharded_local_dev(nranks: int, grid: hj.Grid, model: hj.DynamicsModel,
                            dbounds: hj.IntervalField, init_ptr: int, c_ptr: int, out_ptr: int,
                            cfg: hj.SolveConfig, ctx: hj.Context | None = None,
                            history_capacity: int = 0):
    """hjb_solve_sharded_local_dev: the slab-partitioned solve with `nranks`
    in-process ranks on one device (full-grid device pointers); the same
    per-rank plan, halo offsets and overlap as the NCCL path."""
    lib = abi.load()
    r, rh, wh = hj._c_result(int(history_capacity))
    g, m, d, c = grid.to_c(), model.to_c(), dbounds.to_c(), cfg.to_c()
    hj._check(lib.hjb_solve_sharded_local_dev(hj._ctx(ctx), int(nranks), C.byref(g), C.byref(m),
                                              C.byref(d), C.c_void_p(init_ptr), C.c_void_p(c_ptr),
                                              C.byref(c), C.c_void_p(out_ptr), C.byref(r)))
    n = min(int(r.iterations), int(r.history_capacity))
    return hj.SolveResult(value=None, iterations=int(r.iterations), dt=float(r.dt),
                          wall_seconds=float(r.wall_seconds), converged=bool(r.converged),
                          residual_history=rh[:n].copy(), wall_ms_history=wh[:n].copy(),
                          nodes_per_sweep=int(r.nodes_per_sweep),
                          final_residual=float(r.final_residual))
