"""Row-sharded solve over several GPUs.

A's rows are split over the ranks of a torch.distributed process group
(balanced by nonzeros); every rank also owns a contiguous slice of the
columns (cone-aligned). One iteration of solver.py:313-317 in the reduced
two-pass form becomes

    partial = A_r^T h_r                      column pass over the local rows (all n columns)
    ath_s   = reduce-scatter(partial, sum)   the exchange step (NCCL over NVLink)
    x_s, z_s, delta_s <- column update        x_update / z_update / delta update on the slice,
                                              with GLOBAL column counts (uv.py:82)
    x       = all-gather(x_s)
    lam_r, h_r <- row pass(x)                 y_update + dual updates of the local rows

and every check_every iterations the report parts (row part local, A^T lam via
a second reduce-scatter) are all-reduced and check_termination decides on every
rank identically. Rows never move; the only collectives carry n-vectors.

The compute of a rank is a *backend* (``CudaRankBackend``: libcfb200 kernels
through the C ABI; the CPU tests use a numpy backend with the same interface
on the gloo backend). Parity: the sums over rows of A^T h are split per rank,
so iterates agree with ``solve`` to rounding (not bit for bit).
"""

from __future__ import annotations

import math
from dataclasses import replace

import numpy as np

from .api import IterationReport, SolveResult, SolverConfig, _decide, norms
from .problem import ConeSpec, ProblemInstance, TripletMatrix, cone_sizes_array

__all__ = ["solve_distributed", "choose_sharding", "column_cuts", "row_cuts_from_counts", "exchange_bytes", "solve_sharded", "run_sharded", "partition", "CudaRankBackend", "assemble_report",
           "solve_col_sharded", "run_col_sharded", "CudaColBackend", "local_columns"]

# report parts: row = {sum prim^2, max|prim|, max|Ax|, sum b.lam, nonfinite};
# column = {sum dual^2, max|dual|, sum stat^2, max|stat|, max|A^T lam|, sum c.x, cone_gap, nonfinite}


def partition(p, world: int):
    """Row blocks balanced by nonzeros and cone-aligned column slices of equal-ish size.

    Returns (row_cuts[world+1], col_cuts[world+1])."""
    m, n = int(p.A.num_rows), int(p.A.num_cols)
    row_cuts = row_cuts_from_counts(np.bincount(np.asarray(p.A.rows, dtype=np.int64), minlength=m), world)
    return row_cuts, column_cuts(cone_sizes_array(p.cones), n, world)


def row_cuts_from_counts(counts, world: int):
    """Row blocks balanced by nonzeros from per-row counts (numpy or a device tensor's copy)."""
    counts = np.asarray(counts, dtype=np.int64)
    m = counts.size
    cum = np.concatenate(([0], np.cumsum(counts)))
    cuts = [0] + [int(np.searchsorted(cum, r * cum[-1] / world, side="left")) for r in range(1, world)] + [m]
    return [int(v) for v in np.maximum.accumulate(np.minimum(cuts, m))]


def column_cuts(sizes, n: int, world: int):
    """Cone-aligned column slices of equal-ish size (no cone crosses a slice)."""
    sizes = np.asarray(sizes, dtype=np.int64)
    starts = np.concatenate(([0], np.cumsum(sizes))) if sizes.size else np.array([0, n])
    col_cuts = [0]
    for r in range(1, world):
        k = int(np.searchsorted(starts, r * n / world, side="left"))
        col_cuts.append(int(starts[min(k, len(starts) - 1)]))
    col_cuts.append(n)
    return [int(v) for v in np.maximum.accumulate(np.minimum(col_cuts, n))]


def local_problem(p, r0: int, r1: int):
    """The rank's rows [r0, r1) renumbered from 0, all columns (cones do not matter to the row block)."""
    rows = np.asarray(p.A.rows, dtype=np.int64)
    sel = (rows >= r0) & (rows < r1)
    a = TripletMatrix._view(r1 - r0, p.A.num_cols, rows[sel] - r0, np.asarray(p.A.cols, dtype=np.int64)[sel],
                            np.asarray(p.A.vals, dtype=np.float64)[sel])   # fresh arrays already: no second copy
    return ProblemInstance._view(a, np.ascontiguousarray(np.asarray(p.b, dtype=np.float64)[r0:r1]),
                                 np.asarray(p.c, dtype=np.float64), ConeSpec.orthant(p.A.num_cols))


def assemble_report(k: int, f: list) -> IterationReport:
    """compute_report's final assembly (solver.py:219-242) from the reduced parts."""
    prim2, prim_inf, ax_inf, blam, nf_row, dual2, dual_inf, stat2, stat_inf, atl_inf, pobj, cone_gap, nf_col = f
    return IterationReport(
        iter=k, prim_res_inf=prim_inf, prim_res_2=math.sqrt(prim2), dual_res_inf=dual_inf,
        dual_res_2=math.sqrt(dual2), stat_res_inf=stat_inf, stat_res_2=math.sqrt(stat2), ax_inf=ax_inf,
        atl_inf=atl_inf, cone_gap=cone_gap, pobj=pobj, dobj=-blam, gap=pobj + blam,
        status="diverged" if (nf_row > 0 or nf_col > 0) else "running",
    )


class _DevArray:
    """Zero-copy torch view of a device buffer owned by a cf_plan."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


def torch_all_ranks(torch, flag: bool, group, device) -> bool:
    """True on every rank iff ``flag`` is true on every rank."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return flag
    t = torch.tensor([1.0 if flag else 0.0], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(t.item() > 0)


def _mc_create_export(L, size, world, mc):
    import ctypes

    from . import _lib

    fd = ctypes.c_int(-1)
    _lib.check(L.cf_mc_create(size, world, ctypes.byref(mc), ctypes.byref(fd)))
    return fd.value


def _share_fd(make_fd, rank, group):
    """Rank 0 runs make_fd() and passes the descriptor to every other rank of the (single-node)
    group over an abstract Unix socket (SCM_RIGHTS); returns the descriptor on every rank."""
    import os
    import socket
    import uuid

    import torch.distributed as dist

    world = dist.get_world_size(group)
    name = [None]
    if rank == 0:
        name[0] = "\0cfb200-nvls-" + uuid.uuid4().hex
    dist.broadcast_object_list(name, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    if rank == 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name[0])
        srv.listen(world)
        fd = make_fd()
        dist.barrier(group=group)                      # the others connect after the listen
        for _ in range(world - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"fd"], [fd])
            conn.close()
        srv.close()
        dist.barrier(group=group)
        return fd
    dist.barrier(group=group)
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    cli.connect(name[0])
    _, fds, _, _ = socket.recv_fds(cli, 16, 1)
    cli.close()
    dist.barrier(group=group)
    return fds[0]


class CudaRankBackend:
    """One rank on its GPU: a plan over its row block (all columns) + its column slice state."""

    def __init__(self, lp, col_lo: int, col_hi: int, cone_ptr_slice, global_counts_slice_fn, plan=None,
                 c_slice=None):
        import ctypes

        import torch

        from . import _lib
        from .engine import DevicePlan

        self.torch = torch
        self.lib = _lib.lib()
        self.stream = torch.cuda.current_stream()
        self.plan = plan if plan is not None else DevicePlan.from_problem(lp, stream=self.stream.cuda_stream)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.n, self.m = self.plan.n, self.plan.m
        self.lo, self.hi = col_lo, col_hi

        def view(which):
            ptr, ln = ctypes.c_void_p(), ctypes.c_int64()
            _lib.check(self.lib.cf_plan_vector(self.plan.handle, which, ctypes.byref(ptr), ctypes.byref(ln)))
            return torch.as_tensor(_DevArray(ptr.value or 0, ln.value), device=self.device) if ln.value else \
                torch.zeros(0, dtype=torch.float64, device=self.device)

        self.x_full, self.lam, self.h = view(0), view(3), view(4)
        self.partial = torch.zeros(self.n, dtype=torch.float64, device=self.device)
        ns = col_hi - col_lo
        self.xs = torch.zeros(ns, dtype=torch.float64, device=self.device)
        self.zs = torch.zeros_like(self.xs)
        self.ds = torch.zeros_like(self.xs)
        if c_slice is not None:
            self.cs = c_slice
        else:
            self.cs = torch.as_tensor(np.array(np.asarray(lp.c)[col_lo:col_hi]), dtype=torch.float64,
                                      device=self.device)
        cnt = torch.zeros(self.n, dtype=torch.float64, device=self.device)
        _lib.check(self.lib.cf_plan_column_counts(self.plan.handle, ctypes.c_void_p(cnt.data_ptr())))
        self.local_counts = cnt
        self.cnt_s = None   # set by the driver after the all-reduce of the counts
        self.cone_ptr = None if cone_ptr_slice is None else torch.as_tensor(cone_ptr_slice, dtype=torch.int32,
                                                                            device=self.device)
        self.n_blocks = 0 if cone_ptr_slice is None else len(cone_ptr_slice) - 1

    def _p(self, t):
        import ctypes

        return ctypes.c_void_p(t.data_ptr()) if t.numel() else ctypes.c_void_p(0)

    def partial_At(self, which: str):
        vec = self.h if which == "h" else self.lam
        if self.m == 0:
            self.partial.zero_()
        else:
            self.plan.apply_At(vec.data_ptr(), self.partial.data_ptr())
        return self.partial

    def partial_range_into(self, which: str, out, col_lo: int, col_hi: int):
        """The column tiles of A^T (h or lam) that start in [col_lo, col_hi), into out (no host sync)."""
        vec = self.h if which == "h" else self.lam
        if self.m == 0:
            out[col_lo:col_hi].zero_()
        else:
            from . import _lib

            _lib.check(self.lib.cf_apply_At_cols(self.plan.handle, self._p(vec), self._p(out), int(col_lo),
                                                 int(col_hi)))

    def partial_into(self, which: str, out):
        """A^T (h or lam) of the local rows straight into `out` (n doubles), no host sync."""
        vec = self.h if which == "h" else self.lam
        if self.m == 0:
            out.zero_()
        else:
            from . import _lib

            _lib.check(self.lib.cf_apply_At_async(self.plan.handle, self._p(vec), self._p(out)))

    @classmethod
    def from_plan(cls, plan, col_lo: int, col_hi: int, c_slice, cone_ptr_slice=None):
        """A rank backend over a plan already built on the device (devgen.generate_device_shard)."""
        return cls(None, col_lo, col_hi, cone_ptr_slice, None, plan=plan, c_slice=c_slice)

    def column_update(self, ath_s, mu: float):
        from . import _lib

        _lib.check(self.lib.cf_column_update(self.xs.numel(), self._p(ath_s), self._p(self.cnt_s), self._p(self.cs),
                                             self._p(self.xs), self._p(self.zs), self._p(self.ds), float(mu),
                                             self.n_blocks, self._p(self.cone_ptr) if self.cone_ptr is not None
                                             else None, self.stream.cuda_stream))

    # -------------------------------------------------------------- fused P2P step
    def enable_p2p(self, group, col_cuts):
        """Peer buffers for the fused step: this rank's partial A^T h and x replica live in
        cudaMalloc'ed, IPC-exported memory; every rank opens every other rank's pair. The plan
        then runs on the replica (cf_plan_bind_x), which peers fill with their x+ slices."""
        import ctypes

        import torch.distributed as dist

        from . import _lib

        if getattr(self, "_p2p_own", None):
            return
        self._p2p_group = group
        torch = self.torch
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        self._p2p_own, handles = [], []
        for _ in range(2):   # partial, x replica
            ptr, h = ctypes.c_void_p(), ctypes.create_string_buffer(64)
            _lib.check(self.lib.cf_ipc_alloc(8 * max(self.n, 1), ctypes.byref(ptr), h))
            self._p2p_own.append(ptr.value)
            handles.append(h.raw)
        everyone = [None] * world
        if world > 1:
            dist.all_gather_object(everyone, handles, group=group)
        else:
            everyone = [handles]
        self._p2p_opened = []
        peers = []
        for s in range(world):
            if s == rank:
                peers.append(tuple(self._p2p_own))
                continue
            pair = []
            for h in everyone[s]:
                ptr = ctypes.c_void_p()
                _lib.check(self.lib.cf_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(ptr)))
                self._p2p_opened.append(ptr.value)
                pair.append(ptr.value)
            peers.append(tuple(pair))
        off = 8 * self.lo
        self.p2p_parts = torch.tensor([peers[s][0] + off for s in range(world)], dtype=torch.int64,
                                      device=self.device)
        self.p2p_xdst = torch.tensor([peers[s][1] + off for s in range(world)], dtype=torch.int64,
                                     device=self.device)
        self.p2p_world = world
        self.p2p_partial = torch.as_tensor(_DevArray(self._p2p_own[0], self.n), device=self.device)
        _lib.check(self.lib.cf_plan_bind_x(self.plan.handle, ctypes.c_void_p(self._p2p_own[1])))
        self.x_full = torch.as_tensor(_DevArray(self._p2p_own[1], self.n), device=self.device)

    def column_update_p2p(self, mu: float):
        """Reduce (rank-order sum of the peers' partials) + column update + broadcast of x+
        to every replica, one kernel (cf_column_update_p2p)."""
        from . import _lib

        _lib.check(self.lib.cf_column_update_p2p(
            self.xs.numel(), self._p(self.p2p_parts), self.p2p_world, self._p(self.cnt_s), self._p(self.cs),
            self._p(self.xs), self._p(self.zs), self._p(self.ds), float(mu), self.n_blocks,
            self._p(self.cone_ptr) if self.cone_ptr is not None else None, self._p(self.p2p_xdst), self.p2p_world,
            self.stream.cuda_stream))

    def x_replica(self):
        """This rank's full x (torch), filled by every rank's fused step."""
        return self.x_full

    # ------------------------------------------------------------ NVLS (NVLink SHARP) step
    def enable_nvls(self, group, col_cuts):
        """One multicast object (cf_mc_*) per team holding [partial A^T h | x replica | barrier
        counter], one physical copy per rank. The fused step reads the partials' SUM with
        multimem.ld_reduce and writes x+ into every replica with multimem.st; the barrier is a
        device-side multimem counter. world > 1: rank 0 creates the object and hands its
        POSIX fd to the other ranks over a Unix socket."""
        import ctypes

        import torch.distributed as dist

        from . import _lib

        if getattr(self, "_mc", None):
            return
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        L = self.lib
        sup = ctypes.c_int(0)
        _lib.check(L.cf_mc_supported(ctypes.byref(sup)))
        ok = torch_all_ranks(self.torch, bool(sup.value), group, self.device)
        if not ok:
            raise RuntimeError("NVLS: multicast objects are not supported on every rank's device")
        seg = -(-(8 * max(self.n, 1) + 64) // 256) * 256
        size = 2 * seg + 256
        mc = ctypes.c_void_p()
        if world == 1:
            _lib.check(L.cf_mc_create(size, 1, ctypes.byref(mc), None))
        else:
            fd = _share_fd(lambda: _mc_create_export(L, size, world, mc), rank, group)
            if rank != 0:
                _lib.check(L.cf_mc_import(fd, size, world, ctypes.byref(mc)))
        self._mc = mc.value
        self._mc_group = group
        _lib.check(L.cf_mc_add_device(ctypes.c_void_p(self._mc)))
        uc, mcp = ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(L.cf_mc_bind(ctypes.c_void_p(self._mc), ctypes.byref(uc), ctypes.byref(mcp)))
        if world > 1:
            dist.barrier(group=group)
        self._mc_uc, self._mc_mc = uc.value, mcp.value
        self.nvls_partial = self.torch.as_tensor(_DevArray(self._mc_uc, self.n), device=self.device)
        self._nvls_parts_mc = self._mc_mc + 8 * self.lo
        self._nvls_x_mc = self._mc_mc + seg + 8 * self.lo
        self._nvls_flag_uc, self._nvls_flag_mc = self._mc_uc + 2 * seg, self._mc_mc + 2 * seg
        self._nvls_world, self._nvls_epoch = world, 0
        _lib.check(L.cf_plan_bind_x(self.plan.handle, ctypes.c_void_p(self._mc_uc + seg)))
        self.x_full = self.torch.as_tensor(_DevArray(self._mc_uc + seg, self.n), device=self.device)

    def nvls_barrier(self):
        """Stream-ordered team barrier on the multicast counter (cf_mc_barrier)."""
        import ctypes

        from . import _lib

        self._nvls_epoch += 1
        _lib.check(self.lib.cf_mc_barrier(ctypes.c_void_p(self._nvls_flag_mc), ctypes.c_void_p(self._nvls_flag_uc),
                                          self._nvls_world * self._nvls_epoch, self.stream.cuda_stream))

    def column_update_nvls(self, mu: float):
        """The switch sums the ranks' partials (multimem.ld_reduce), then the column update,
        then x+ into every replica (multimem.st): cf_column_update_nvls."""
        import ctypes

        from . import _lib

        _lib.check(self.lib.cf_column_update_nvls(
            self.xs.numel(), ctypes.c_void_p(self._nvls_parts_mc), self._p(self.cnt_s), self._p(self.cs),
            self._p(self.xs), self._p(self.zs), self._p(self.ds), float(mu), self.n_blocks,
            self._p(self.cone_ptr) if self.cone_ptr is not None else None, ctypes.c_void_p(self._nvls_x_mc),
            self.stream.cuda_stream))

    def disable_nvls(self):
        import ctypes

        import torch.distributed as dist

        from . import _lib

        if not getattr(self, "_mc", None):
            return
        self.torch.cuda.synchronize()
        _lib.check(self.lib.cf_plan_bind_x(self.plan.handle, None))
        if dist.is_available() and dist.is_initialized():
            dist.barrier(group=getattr(self, "_mc_group", None))   # no peer still stores into our copy
        self.lib.cf_mc_destroy(ctypes.c_void_p(self._mc))
        self._mc = None
        ptr, ln = ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(self.lib.cf_plan_vector(self.plan.handle, 0, ctypes.byref(ptr), ctypes.byref(ln)))
        self.x_full = self.torch.as_tensor(_DevArray(ptr.value or 0, ln.value), device=self.device)


    def disable_p2p(self):
        import ctypes

        if not getattr(self, "_p2p_own", None):
            return
        from . import _lib

        self.torch.cuda.synchronize()
        _lib.check(self.lib.cf_plan_bind_x(self.plan.handle, None))
        for ptr in self._p2p_opened:
            self.lib.cf_ipc_close(ctypes.c_void_p(ptr))
        # every peer must have closed its mapping of our buffers before we free them (freeing
        # exported memory before the importer's cudaIpcCloseMemHandle is undefined)
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            dist.barrier(group=getattr(self, "_p2p_group", None))
        for ptr in self._p2p_own:
            self.lib.cf_ipc_free(ctypes.c_void_p(ptr))
        self._p2p_own, self._p2p_opened = [], []
        ptr, ln = ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(self.lib.cf_plan_vector(self.plan.handle, 0, ctypes.byref(ptr), ctypes.byref(ln)))
        self.x_full = self.torch.as_tensor(_DevArray(ptr.value or 0, ln.value), device=self.device)

    def x_slice(self):
        return self.xs

    def set_x(self, x_full):
        self.x_full.copy_(x_full)

    def row_step(self, mu: float, report: bool):
        from . import _lib

        _lib.check(self.lib.cf_plan_row_step(self.plan.handle, float(mu), 1 if report else 0))

    def row_parts(self):
        from . import _lib

        out = np.zeros(5)
        _lib.check(self.lib.cf_plan_row_parts(self.plan.handle, self._np(out)))
        return out

    def col_parts(self, atl_s):
        from . import _lib

        out = np.zeros(8)
        _lib.check(self.lib.cf_column_parts(self.xs.numel(), self._p(atl_s), self._p(self.cs), self._p(self.xs),
                                            self._p(self.zs), self._p(self.ds), self._np(out),
                                            self.stream.cuda_stream))
        return out

    @staticmethod
    def _np(a):
        import ctypes

        return ctypes.c_void_p(a.ctypes.data)

    def lam_local(self):
        return self.lam

    def close(self):
        self.disable_p2p()
        self.disable_nvls()
        self.plan.close()


def _cone_ptr_slice(p, lo: int, hi: int):
    sizes = cone_sizes_array(p.cones)
    if sizes.size == 0 or int(sizes.max()) == 1:
        return None
    starts = np.concatenate(([0], np.cumsum(sizes)))
    q0, q1 = np.searchsorted(starts, lo), np.searchsorted(starts, hi)
    return (starts[q0:q1 + 1] - lo).astype(np.int32)


def solve_sharded(p, cfg: SolverConfig | None = None, group=None, backend_factory=None,
                  p2p: bool = False, nvls: bool = False) -> SolveResult:
    """solve() with A's rows split over the ranks of ``group`` (every rank passes the same problem).

    Cold start only. Returns the same SolveResult on every rank. ``p2p``: the fused
    peer-memory step (run_sharded) instead of NCCL reduce-scatter + all-gather."""
    import torch.distributed as dist

    cfg = cfg or SolverConfig()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    row_cuts, col_cuts = partition(p, world)
    r0, r1 = row_cuts[rank], row_cuts[rank + 1]
    lo, hi = col_cuts[rank], col_cuts[rank + 1]
    lp = local_problem(p, r0, r1)
    factory = backend_factory or CudaRankBackend
    be = factory(lp, lo, hi, _cone_ptr_slice(p, lo, hi), None)
    try:
        return run_sharded(be, row_cuts, col_cuts, cfg, norms(p.b), norms(p.c), group, p2p=p2p, nvls=nvls)
    finally:
        if hasattr(be, "close"):
            be.close()


def run_sharded(be, row_cuts, col_cuts, cfg, b_norms, c_norms, group=None, timing=None,
                gather_result: bool = True, overlap_reduce: bool = True, p2p: bool = False,
                nvls: bool = False) -> SolveResult:
    """The sharded loop on an existing rank backend (row/column cuts shared by all ranks).

    ``timing``: if a dict, receives the CUDA-event time of the loop on this rank (ms).
    ``overlap_reduce``: NCCL + CUDA backend: reduce A^T h slice by slice, overlapped with the
    next slice's column pass (else one reduce-scatter after the whole pass).
    ``p2p``: CUDA backend: the fused step instead. A^T h is computed into peer-visible memory,
    then a barrier, then one kernel per rank that sums its slice over the peers in rank order,
    updates it and stores x+ into every rank's x replica over NVLink, then a barrier. That
    replaces the reduce-scatter, the column update and the all-gather.
    ``nvls``: the same fused step with the reduction and the broadcast done by the NVSwitch
    (multimem.ld_reduce / multimem.st on a multicast object, enable_nvls) and a device-side
    multimem counter as the barrier."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = col_cuts[rank], col_cuts[rank + 1]
    torch_dev = be.device
    n = col_cuts[-1]
    S = max(col_cuts[r + 1] - col_cuts[r] for r in range(world))
    Mx = max(row_cuts[r + 1] - row_cuts[r] for r in range(world))
    contiguous = all(col_cuts[r] == r * S for r in range(world))
    nccl = dist.get_backend(group) == "nccl"
    padded = torch.zeros(world * S, dtype=torch.float64, device=torch_dev)
    rs_out = torch.empty(S, dtype=torch.float64, device=torch_dev)
    ag_out = torch.empty(world * S, dtype=torch.float64, device=torch_dev)
    xs_pad = torch.zeros(S, dtype=torch.float64, device=torch_dev)
    pad_idx = None
    if not contiguous:
        # slice r at [r*S, r*S + len_r) of the padded layout
        pad_idx = torch.cat([torch.arange(col_cuts[r], col_cuts[r + 1], dtype=torch.int64) - col_cuts[r] + r * S
                             for r in range(world)]).to(torch_dev)

    # NCCL fast path: A^T h lands directly in the reduce-scatter input and x is
    # all-gathered straight into the plan's x buffer (no staging copies, no host sync)
    fast = (nccl and contiguous and hasattr(be, "partial_into") and world * S == n
            and getattr(be, "xs", None) is not None and be.xs.numel() == S)

    # overlap: the column pass runs slice by slice (tiles starting in slice r); slice r's
    # sums go to their owner with an async NCCL reduce while slice r+1 computes
    overlap = fast and overlap_reduce and hasattr(be, "partial_range_into")

    def reduce_scatter_partial(which):
        if not fast:
            return reduce_scatter(be.partial_At(which))
        if overlap:
            works = []
            for r in range(world):
                be.partial_range_into(which, padded, col_cuts[r], col_cuts[r + 1])
                dst = r if group is None else dist.get_global_rank(group, r)
                works.append(dist.reduce(padded[col_cuts[r]:col_cuts[r + 1]], dst=dst, op=dist.ReduceOp.SUM,
                                         group=group, async_op=True))
            for w in works:
                w.wait()
            return padded[lo:hi]
        be.partial_into(which, padded)
        dist.reduce_scatter_tensor(rs_out, padded, op=dist.ReduceOp.SUM, group=group)
        return rs_out

    def reduce_scatter(vec):
        if contiguous:
            padded[:n].copy_(vec)
        else:
            padded[pad_idx] = vec
        if nccl:
            dist.reduce_scatter_tensor(rs_out, padded, op=dist.ReduceOp.SUM, group=group)
            out = rs_out
        else:
            dist.all_reduce(padded, op=dist.ReduceOp.SUM, group=group)
            out = padded[rank * S:(rank + 1) * S]
        return out[:hi - lo].contiguous()

    def gather_x(slice_vec):
        xs_pad[:slice_vec.numel()] = slice_vec
        if nccl:
            dist.all_gather_into_tensor(ag_out, xs_pad, group=group)
        else:
            parts = list(ag_out.chunk(world))
            dist.all_gather(parts, xs_pad, group=group)
            ag_out.copy_(torch.cat(parts))
        return ag_out[:n] if contiguous else ag_out[pad_idx]

    use_nvls = nvls and hasattr(be, "enable_nvls")
    if nvls and not use_nvls:
        raise ValueError("nvls=True needs a backend with enable_nvls")
    use_p2p = (not use_nvls) and p2p and hasattr(be, "enable_p2p") and hasattr(be, "partial_into")
    bar = torch.zeros(1, dtype=torch.float64, device=torch_dev)

    def barrier():
        # stream-ordered cross-rank barrier: the all-reduce finishes on any rank only after
        # every rank's earlier work on its stream (partials written / replicas filled)
        if world > 1:
            dist.all_reduce(bar, group=group)

    # global column counts (uv.py:82 uses counts over ALL rows)
    be.cnt_s = reduce_scatter(be.local_counts).clone()
    if use_p2p:
        be.enable_p2p(group, col_cuts)
    if use_nvls:
        be.enable_nvls(group, col_cuts)
    trace = []
    x_full = None
    if timing is not None and torch_dev.type == "cuda":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
    for k in range(1, cfg.max_iters + 1):
        if use_nvls:
            be.partial_into("h", be.nvls_partial)
            be.nvls_barrier()
            be.column_update_nvls(cfg.mu)
            be.nvls_barrier()
            x_full = be.x_replica()
        elif use_p2p:
            be.partial_into("h", be.p2p_partial)
            barrier()
            be.column_update_p2p(cfg.mu)
            barrier()
            x_full = be.x_replica()
        else:
            ath = reduce_scatter_partial("h")
            be.column_update(ath, cfg.mu)
        if use_p2p or use_nvls:
            pass
        elif fast:
            dist.all_gather_into_tensor(be.x_full, be.xs, group=group)
            x_full = be.x_full
        else:
            x_full = gather_x(be.x_slice())
            be.set_x(x_full)
        report = (k % cfg.check_every == 0) or (k == cfg.max_iters)
        be.row_step(cfg.mu, report)
        if not report:
            continue
        rp = torch.as_tensor(be.row_parts(), dtype=torch.float64, device=torch_dev)
        atl = reduce_scatter_partial("lam")
        cp = torch.as_tensor(be.col_parts(atl), dtype=torch.float64, device=torch_dev)
        sums = torch.stack([rp[0], rp[3], cp[0], cp[2], cp[5]])
        maxs = torch.stack([rp[1], rp[2], rp[4], cp[1], cp[3], cp[4], cp[6], cp[7]])
        nan = torch.isnan(maxs).to(torch.float64)
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(maxs, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(nan, op=dist.ReduceOp.MAX, group=group)
        maxs = torch.where(nan > 0, torch.full_like(maxs, float("nan")), maxs)
        s, mx = sums.tolist(), maxs.tolist()
        f = [s[0], mx[0], mx[1], s[1], mx[2], s[2], mx[3], s[3], mx[4], mx[5], s[4], mx[6], mx[7]]
        rep = assemble_report(k, f)
        status = _decide(rep, cfg, b_norms, c_norms)
        if status == "running" and k == cfg.max_iters:
            status = "max_iters"
        trace.append(replace(rep, status=status))
        if status != "running":
            break
    if timing is not None and torch_dev.type == "cuda":
        e1.record()
        e1.synchronize()
        timing["loop_ms"] = e0.elapsed_time(e1)
        timing["iters"] = trace[-1].iter
    if not gather_result:
        return SolveResult(x=None, lam=None, report=trace[-1], trace=tuple(trace))
    lam_pad = torch.zeros(Mx, dtype=torch.float64, device=torch_dev)
    lam_local = be.lam_local()
    lam_pad[:lam_local.numel()] = lam_local
    parts = [torch.empty(Mx, dtype=torch.float64, device=torch_dev) for _ in range(world)]
    dist.all_gather(parts, lam_pad, group=group)
    lam = torch.cat([parts[r][:row_cuts[r + 1] - row_cuts[r]] for r in range(world)])
    return SolveResult(x=x_full.detach().cpu().numpy().copy(), lam=lam.detach().cpu().numpy().copy(),
                       report=trace[-1], trace=tuple(trace))


# ------------------------------------------------------------------ column sharding
# SURVEY §8e alternative for m < n: every rank holds A's columns [lo, hi) with ALL rows.
# One iteration is
#
#     x_s, z_s, delta_s <- column pass on the slice (h is full and local)
#     ax   = all-reduce(A_s x_s, sum)            the only exchange: one m-vector
#     lam, h <- row update of every row from ax   (the same on every rank)
#
# so a rank sends ~2m(p-1)/p doubles per iteration instead of the row-sharded 2n(p-1)/p.
# Reports: the row part is computed locally from the full vectors (identical on every
# rank); the column part (A_s^T lam over the slice) is all-reduced.

def local_columns(p, c0: int, c1: int):
    """The rank's columns [c0, c1) renumbered from 0, all rows, with the slice's cones.

    Entries already sorted by column (canonical order, as generate.py stores them) are a
    contiguous range found by binary search; any other order takes a mask pass."""
    cols = np.asarray(p.A.cols, dtype=np.int64)
    if cols.size and bool(np.all(cols[1:] >= cols[:-1])):
        k0, k1 = int(np.searchsorted(cols, c0, "left")), int(np.searchsorted(cols, c1, "left"))
        sel = slice(k0, k1)
    else:
        sel = (cols >= c0) & (cols < c1)
    # views where possible (no copy of the caller's 100M-entry arrays: the plan copies them to the GPU)
    rows = np.ascontiguousarray(np.asarray(p.A.rows, dtype=np.int64)[sel])
    vals = np.ascontiguousarray(np.asarray(p.A.vals, dtype=np.float64)[sel])
    lcols = np.ascontiguousarray(cols[sel]) if c0 == 0 else cols[sel] - c0
    a = TripletMatrix._view(p.A.num_rows, c1 - c0, rows, lcols, vals)
    sizes = cone_sizes_array(p.cones)
    starts = np.concatenate(([0], np.cumsum(sizes)))
    q0, q1 = int(np.searchsorted(starts, c0)), int(np.searchsorted(starts, c1))
    return ProblemInstance._view(a, np.asarray(p.b, dtype=np.float64), np.ascontiguousarray(np.asarray(p.c, dtype=np.float64)[c0:c1]),
                                 ConeSpec(sizes[q0:q1]))


class CudaColBackend:
    """One rank of the column-sharded solve: a plan over its column slice (all rows)."""

    def __init__(self, lp, plan=None):
        import ctypes

        import torch

        from . import _lib
        from .engine import DevicePlan

        self.torch = torch
        self.lib = _lib.lib()
        self.stream = torch.cuda.current_stream()
        self.plan = plan if plan is not None else DevicePlan.from_problem(lp, stream=self.stream.cuda_stream)
        self.plan.set_state(1.0, None, export=False)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.m, self.n = self.plan.m, self.plan.n

        def view(which):
            ptr, ln = ctypes.c_void_p(), ctypes.c_int64()
            _lib.check(self.lib.cf_plan_vector(self.plan.handle, which, ctypes.byref(ptr), ctypes.byref(ln)))
            return torch.as_tensor(_DevArray(ptr.value or 0, ln.value), device=self.device) if ln.value else \
                torch.zeros(0, dtype=torch.float64, device=self.device)

        self.x, self.z, self.delta, self.lam, self.ax, self.c = view(0), view(1), view(2), view(3), view(5), view(7)
        self.atl = torch.zeros(self.n, dtype=torch.float64, device=self.device)

    @staticmethod
    def _p(t):
        import ctypes

        return ctypes.c_void_p(t.data_ptr()) if t.numel() else ctypes.c_void_p(0)

    def row_norms(self):
        """(d, amax) of the slice's entries per row, device tensors of m."""
        from . import _lib

        d = self.torch.zeros(self.m, dtype=self.torch.float64, device=self.device)
        am = self.torch.zeros(self.m, dtype=self.torch.float64, device=self.device)
        _lib.check(self.lib.cf_plan_row_norms(self.plan.handle, self._p(d), self._p(am)))
        return d, am

    def set_row_norms(self, d, am):
        from . import _lib

        _lib.check(self.lib.cf_plan_set_row_norms(self.plan.handle, self._p(d), self._p(am)))

    def col_step(self, mu: float):
        from . import _lib

        _lib.check(self.lib.cf_plan_col_step(self.plan.handle, float(mu)))

    def partial_Ax(self):
        """A_s x_s into the plan's ax buffer (the driver all-reduces it in place)."""
        from . import _lib

        if self.n:
            _lib.check(self.lib.cf_apply_A_async(self.plan.handle, self._p(self.x), self._p(self.ax)))
        else:
            self.ax.zero_()
        return self.ax

    def row_update(self, mu: float, report: bool):
        from . import _lib

        _lib.check(self.lib.cf_plan_row_update(self.plan.handle, float(mu), 1 if report else 0))

    def row_parts(self):
        from . import _lib

        out = np.zeros(5)
        _lib.check(self.lib.cf_plan_row_parts(self.plan.handle, ctypes_ptr(out)))
        return out

    def col_parts(self):
        from . import _lib

        out = np.zeros(8)
        if self.n:
            _lib.check(self.lib.cf_apply_At_async(self.plan.handle, self._p(self.lam), self._p(self.atl)))
        _lib.check(self.lib.cf_column_parts(self.n, self._p(self.atl), self._p(self.c), self._p(self.x),
                                            self._p(self.z), self._p(self.delta), ctypes_ptr(out),
                                            self.stream.cuda_stream))
        return out

    def x_slice(self):
        return self.x

    def lam_full(self):
        return self.lam

    # ---- the sharded row update (run_col_sharded shard_rows)
    def ax_into(self, out):
        """A_s x_s into out[:m] (out: the padded reduce-scatter input)."""
        from . import _lib

        if self.n:
            _lib.check(self.lib.cf_apply_A_async(self.plan.handle, self._p(self.x), self._p(out)))
        else:
            out[:self.m].zero_()

    def bind_h(self, h):
        """Run the column pass on h (the all-gather target), or back on the plan's own (None)."""
        import ctypes

        from . import _lib

        _lib.check(self.lib.cf_plan_bind_h(self.plan.handle, None if h is None else ctypes.c_void_p(h.data_ptr())))

    def row_update_range(self, mu, report, r0, r1, ax_slice):
        from . import _lib

        _lib.check(self.lib.cf_plan_row_update_range(self.plan.handle, float(mu), 1 if report else 0, int(r0), int(r1),
                                                     self._p(ax_slice)))

    def row_parts_range(self, r0, r1, ax_slice):
        from . import _lib

        out = np.zeros(5)
        _lib.check(self.lib.cf_plan_row_parts_range(self.plan.handle, int(r0), int(r1), self._p(ax_slice),
                                                    ctypes_ptr(out)))
        return out

    def lam_range(self, r0, r1):
        return self.lam[r0:r1]

    def set_lam(self, lam_full):
        self.lam.copy_(lam_full)

    def close(self):
        self.plan.close()


def ctypes_ptr(a):
    import ctypes

    return ctypes.c_void_p(a.ctypes.data)


def run_col_sharded(be, col_cuts, cfg, b_norms, c_norms, group=None, timing=None,
                    gather_result: bool = True, shard_rows: bool | None = None) -> SolveResult:
    """The column-sharded loop on an existing rank backend (column cuts shared by all ranks).

    ``shard_rows`` (default: when the backend supports it): instead of all-reducing A x and
    updating every row on every rank, reduce-scatter A x, update this rank's block of
    rows only, and all-gather h (the column passes gather it) — the same NVLink volume as
    the all-reduce, 1/N of the row update's HBM traffic per rank. lam is all-gathered on
    report iterations (A^T lam) and at the end."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    if shard_rows is None:
        shard_rows = hasattr(be, "row_update_range")
    # fu = 1/(1 + d) and the implicit-y finiteness check need WHOLE rows: sum the slices' d
    # (uv.py:81; the association of the sum differs from one GPU's only by rounding)
    d, am = be.row_norms()
    dist.all_reduce(d, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(am, op=dist.ReduceOp.MAX, group=group)
    be.set_row_norms(d, am)
    m = int(d.numel())
    S = -(-m // world) if m else 0
    r0, r1 = min(m, rank * S), min(m, (rank + 1) * S)
    if shard_rows:
        ax_pad = torch.zeros(world * S, dtype=torch.float64, device=be.device)
        h_pad = torch.zeros(world * S + 8, dtype=torch.float64, device=be.device)   # + slack (engine reads)
        be.bind_h(h_pad)
        ax_mine = ax_pad[rank * S:(rank + 1) * S]
        h_mine = h_pad[rank * S:(rank + 1) * S]
        lam_pad = torch.zeros(world * S, dtype=torch.float64, device=be.device)

        def gather_lam():
            lam_pad[rank * S:rank * S + (r1 - r0)] = be.lam_range(r0, r1)
            if nccl:
                dist.all_gather_into_tensor(lam_pad, lam_pad[rank * S:(rank + 1) * S].clone(), group=group)
            else:
                parts = [torch.empty(S, dtype=torch.float64) for _ in range(world)]
                dist.all_gather(parts, lam_pad[rank * S:(rank + 1) * S].clone(), group=group)
                lam_pad.copy_(torch.cat(parts))
            be.set_lam(lam_pad[:m])
    trace = []
    try:   # h stays bound to h_pad only inside the loop (an exception must not leave the plan on it)
        if timing is not None and be.device.type == "cuda":
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        for k in range(1, cfg.max_iters + 1):
            be.col_step(cfg.mu)
            report = (k % cfg.check_every == 0) or (k == cfg.max_iters)
            if shard_rows:
                be.ax_into(ax_pad)
                if nccl:   # in place: this rank's block of the sum lands at its own offset
                    dist.reduce_scatter_tensor(ax_mine, ax_pad, op=dist.ReduceOp.SUM, group=group)
                else:
                    dist.all_reduce(ax_pad, op=dist.ReduceOp.SUM, group=group)
                ax_slice = ax_mine[:r1 - r0]
                be.row_update_range(cfg.mu, report, r0, r1, ax_slice)   # writes h_pad[r0:r1]
                if nccl:
                    dist.all_gather_into_tensor(h_pad[:world * S], h_mine, group=group)
                else:
                    parts = [torch.empty(S, dtype=torch.float64) for _ in range(world)]
                    dist.all_gather(parts, h_mine.clone(), group=group)
                    h_pad[:world * S].copy_(torch.cat(parts))
            else:
                ax = be.partial_Ax()
                dist.all_reduce(ax, op=dist.ReduceOp.SUM, group=group)
                be.row_update(cfg.mu, report)
            if not report:
                continue
            if shard_rows:
                rpl = torch.as_tensor(be.row_parts_range(r0, r1, ax_slice), dtype=torch.float64, device=be.device)
                gather_lam()   # A^T lam below needs every row's lam
            else:
                rpl = None
                rp = be.row_parts()          # full rows: the same on every rank
            cp = torch.as_tensor(be.col_parts(), dtype=torch.float64, device=be.device)
            if shard_rows:   # row parts: {sum prim^2, max|prim|, max|Ax|, sum b.lam, nonfinite} over the blocks
                sums = torch.stack([cp[0], cp[2], cp[5], rpl[0], rpl[3]])
                maxs = torch.stack([cp[1], cp[3], cp[4], cp[6], cp[7], rpl[1], rpl[2], rpl[4]])
            else:
                sums = torch.stack([cp[0], cp[2], cp[5]])
                maxs = torch.stack([cp[1], cp[3], cp[4], cp[6], cp[7]])
            nan = torch.isnan(maxs).to(torch.float64)
            dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
            dist.all_reduce(maxs, op=dist.ReduceOp.MAX, group=group)
            dist.all_reduce(nan, op=dist.ReduceOp.MAX, group=group)
            maxs = torch.where(nan > 0, torch.full_like(maxs, float("nan")), maxs)
            s, mx = sums.tolist(), maxs.tolist()
            if shard_rows:
                rp = [s[3], mx[5], mx[6], s[4], mx[7]]
            f = [rp[0], rp[1], rp[2], rp[3], rp[4], s[0], mx[0], s[1], mx[1], mx[2], s[2], mx[3], mx[4]]
            rep = assemble_report(k, f)
            status = _decide(rep, cfg, b_norms, c_norms)
            if status == "running" and k == cfg.max_iters:
                status = "max_iters"
            trace.append(replace(rep, status=status))
            if status != "running":
                break
        if timing is not None and be.device.type == "cuda":
            e1.record()
            e1.synchronize()
            timing["loop_ms"] = e0.elapsed_time(e1)
            timing["iters"] = trace[-1].iter
        if shard_rows:
            gather_lam()
    finally:
        if shard_rows:
            be.bind_h(None)
    if not gather_result:
        return SolveResult(x=None, lam=None, report=trace[-1], trace=tuple(trace))
    S = max(col_cuts[r + 1] - col_cuts[r] for r in range(world))
    xs = torch.zeros(S, dtype=torch.float64, device=be.device)
    xl = be.x_slice()
    xs[:xl.numel()] = xl
    parts = [torch.empty(S, dtype=torch.float64, device=be.device) for _ in range(world)]
    dist.all_gather(parts, xs, group=group)
    x = torch.cat([parts[r][:col_cuts[r + 1] - col_cuts[r]] for r in range(world)])
    del rank
    return SolveResult(x=x.detach().cpu().numpy().copy(), lam=be.lam_full().detach().cpu().numpy().copy(),
                       report=trace[-1], trace=tuple(trace))


def solve_col_sharded(p, cfg: SolverConfig | None = None, group=None, backend_factory=None,
                      shard_rows: bool | None = None) -> SolveResult:
    """solve() with A's columns split over the ranks of ``group`` (every rank passes the same problem).

    Cold start only. Returns the same SolveResult on every rank."""
    import torch.distributed as dist

    cfg = cfg or SolverConfig()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    col_cuts = column_cuts(cone_sizes_array(p.cones), int(p.A.num_cols), world)   # no row counts needed
    lp = local_columns(p, col_cuts[rank], col_cuts[rank + 1])
    be = (backend_factory or CudaColBackend)(lp)
    try:
        return run_col_sharded(be, col_cuts, cfg, norms(p.b), norms(p.c), group=group, shard_rows=shard_rows)
    finally:
        if hasattr(be, "close"):
            be.close()


def exchange_bytes(m: int, n: int, world: int, mode: str) -> int:
    """NVLink bytes each rank sends per iteration (and receives) for ``mode``.

    rows: reduce-scatter of the n-vector A_r^T h_r plus all-gather of x, 2 * 8n(p-1)/p;
    cols: all-reduce of the m-vector A_s x_s, 2 * 8m(p-1)/p (ring/NVLS volume).
    Reports (every check_every iterations) add one more exchange of the same kind."""
    if world < 1:
        raise ValueError("world must be >= 1")
    if mode == "rows":
        return 2 * 8 * n * (world - 1) // world
    if mode == "cols":
        return 2 * 8 * m * (world - 1) // world
    raise ValueError(f"unknown sharding mode {mode!r}")


def choose_sharding(m: int, n: int, world: int) -> str:
    """Rows or columns for an m x n problem on ``world`` ranks (SURVEY §8e "Alternatives").

    The exchange is the only cross-rank cost of either layout and both keep every
    nonzero on exactly one rank, so the layout that moves fewer bytes wins: column
    sharding when m < n (it all-reduces the m-vector A x), row sharding otherwise
    (it exchanges n-vectors). Ties and world 1 pick rows, the C5 layout."""
    if world <= 1:
        return "rows"
    return "cols" if exchange_bytes(m, n, world, "cols") < exchange_bytes(m, n, world, "rows") else "rows"


def solve_distributed(p, cfg: SolverConfig | None = None, group=None, mode: str = "auto",
                      backend_factory=None, p2p: bool = False) -> SolveResult:
    """solve() over the ranks of ``group`` with the layout picked by ``mode``.

    ``mode``: "auto" (choose_sharding on the problem's shape), "rows" (solve_sharded;
    ``p2p`` selects the fused peer-memory step) or "cols" (solve_col_sharded).
    ``backend_factory`` is the chosen layout's rank backend (CUDA by default). Every
    rank passes the same problem and gets the same SolveResult."""
    import torch.distributed as dist

    if mode not in ("auto", "rows", "cols"):
        raise ValueError(f"unknown sharding mode {mode!r}")
    if mode == "auto":
        mode = choose_sharding(int(p.A.num_rows), int(p.A.num_cols), dist.get_world_size(group))
    if mode == "cols":
        if p2p:
            raise ValueError("p2p is a row-sharding step; column sharding all-reduces A x")
        return solve_col_sharded(p, cfg, group=group, backend_factory=backend_factory)
    return solve_sharded(p, cfg, group=group, backend_factory=backend_factory, p2p=p2p)
