"""Row-sharded solve (C5 path) on CPU: world_size 2 (and 3) over gloo with a numpy rank backend.

The driver (paper_2203_05027_b200/sharded.py: partition, reduce-scatter of the
partial A^T h, sliced column update with global counts, all-gather of x, report
reduction, termination) is the product code; only the per-rank compute is the
numpy test backend below, which restates the CUDA kernels' reduced-form
arithmetic. The sharded result must match the single-process oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from conftest import rel_err

from paper_2203_05027_b200 import GenSpec, SolverConfig, generate
from paper_2203_05027_b200.instances import project_cones_host
from paper_2203_05027_b200.sharded import partition, solve_sharded


class NumpyRankBackend:
    """Test-only restatement of one rank's kernels (cf_column_update / cf_plan_row_step / parts)."""

    def __init__(self, lp, lo, hi, cone_ptr_slice, _unused):
        self.device = torch.device("cpu")
        a = lp.A
        order = np.lexsort((a.rows, a.cols))   # canonical order: bincount sums run in it
        self.rows, self.cols, self.vals = a.rows[order], a.cols[order], a.vals[order]
        self.m, self.n = a.num_rows, a.num_cols
        self.b = np.asarray(lp.b, dtype=np.float64)
        d = np.bincount(self.rows, weights=self.vals * self.vals, minlength=self.m)
        self.fu, self.db = 1.0 / (1.0 + d), d * self.b
        self.lam, self.h, self.ax = np.zeros(self.m), np.zeros(self.m), np.zeros(self.m)
        self.x_full = np.zeros(self.n)
        self.lo, self.hi = lo, hi
        ns = hi - lo
        self.xs, self.zs, self.ds = np.zeros(ns), np.zeros(ns), np.zeros(ns)
        self.cs = np.asarray(lp.c, dtype=np.float64)[lo:hi]
        self.cone_ptr = cone_ptr_slice
        self.local_counts = torch.tensor(np.bincount(self.cols, minlength=self.n).astype(np.float64))
        self.cnt_s = None

    def partial_At(self, which):
        vec = self.h if which == "h" else self.lam
        return torch.tensor(np.bincount(self.cols, weights=self.vals * vec[self.rows], minlength=self.n))

    def column_update(self, ath_s, mu):
        ath, cnt = ath_s.numpy(), self.cnt_s.numpy()
        fv = 1.0 / (1.0 + cnt)
        dm = self.ds / mu
        xp = fv * ((((cnt * self.xs) + ath) + self.zs + dm) - self.cs / mu)
        w = xp - dm
        if self.cone_ptr is None:
            zp = np.where(w > 0.0, w, 0.0)
        else:
            zp = project_cones_host(np.diff(self.cone_ptr).astype(np.int64), w)
        self.ds = self.ds + mu * (zp - xp)
        self.xs, self.zs = xp, zp

    def x_slice(self):
        return torch.tensor(self.xs)

    def set_x(self, x_full):
        self.x_full = x_full.numpy().copy()

    def row_step(self, mu, report):
        ax = np.bincount(self.rows, weights=self.vals * self.x_full[self.cols], minlength=self.m)
        r = self.fu * (self.db + ax)
        self.lam = self.lam + mu * (r - self.b)
        self.h = (self.b - r) - self.lam / mu
        self.ax = ax

    def row_parts(self):
        pr = self.ax - self.b
        if self.m == 0:
            return np.zeros(5)
        return np.array([np.sum(pr * pr), np.max(np.abs(pr)), np.max(np.abs(self.ax)), np.sum(self.b * self.lam),
                         float(not np.isfinite(self.lam).all())])

    def col_parts(self, atl_s):
        atl = atl_s.numpy()
        dual = atl + self.cs
        stat = dual - self.ds
        if atl.size == 0:
            return np.zeros(8)
        return np.array([np.sum(dual * dual), np.max(np.abs(dual)), np.sum(stat * stat), np.max(np.abs(stat)),
                         np.max(np.abs(atl)), np.sum(self.cs * self.xs), np.max(np.abs(self.xs - self.zs)),
                         float(not (np.isfinite(self.xs).all() and np.isfinite(self.zs).all()))])

    def lam_local(self):
        return torch.tensor(self.lam)

    # the fused peer-memory step, with POSIX shared memory standing in for NVLink peer buffers
    def enable_p2p(self, group, col_cuts):
        from multiprocessing import shared_memory

        if getattr(self, "_shm", None):
            return
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        nbytes = 8 * max(self.n, 1)
        self._shm = [shared_memory.SharedMemory(create=True, size=nbytes) for _ in range(2)]
        names = [None] * world
        dist.all_gather_object(names, [s.name for s in self._shm], group=group)
        self._peer_shm = [self._shm if s == rank else [shared_memory.SharedMemory(name=nm) for nm in names[s]]
                          for s in range(world)]
        self._peers = [[np.ndarray((self.n,), np.float64, buffer=s.buf) for s in pair] for pair in self._peer_shm]
        own_partial, own_x = self._peers[rank]
        own_x[:] = self.x_full
        self.p2p_partial = torch.from_numpy(own_partial)
        self.x_full = own_x                       # row_step reads the replica the peers fill
        self.x_full_t = torch.from_numpy(own_x)

    def x_replica(self):
        return self.x_full_t

    def partial_into(self, which, out):
        out.copy_(self.partial_At(which))

    def column_update_p2p(self, mu):
        lo, hi = self.lo, self.hi
        ath = self._peers[0][0][lo:hi].copy()
        for s in range(1, len(self._peers)):
            ath = ath + self._peers[s][0][lo:hi]          # rank order, as cf_column_update_p2p
        self.column_update(torch.from_numpy(ath), mu)
        for pair in self._peers:
            pair[1][lo:hi] = self.xs                     # x+ into every replica

    # the NVLS step: the switch's reduction and broadcast emulated on the same shared memory
    # (the reduction order inside a switch is the hardware's; here rank order)
    def enable_nvls(self, group, col_cuts):
        self.enable_p2p(group, col_cuts)
        self.nvls_partial = self.p2p_partial
        self._nvls_group = group

    def nvls_barrier(self):
        dist.barrier(group=self._nvls_group)

    def column_update_nvls(self, mu):
        self.column_update_p2p(mu)

    def close(self):
        self.x_full = np.array(self.x_full)
        self.p2p_partial = self.x_full_t = None
        self._peers = None
        for pair in getattr(self, "_peer_shm", []) or []:
            for s in pair:
                s.close()
        for s in getattr(self, "_shm", []) or []:
            s.unlink()
        self._shm = self._peer_shm = None


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, spec, cfg_kw, out_path, p2p=False, nvls=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = generate(spec)
        cfg = SolverConfig(**cfg_kw)

        res = solve_sharded(p, cfg, backend_factory=NumpyRankBackend, p2p=p2p, nvls=nvls)
        if rank == 0:
            np.savez(out_path, x=res.x, lam=res.lam, iters=np.array([r.iter for r in res.trace]),
                     status=np.array([r.status for r in res.trace]),
                     pobj=np.array([r.pobj for r in res.trace]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,spec,cfg_kw,mode", [
    (2, GenSpec(40, 90, 0.06, "lp", seed=31), dict(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=4000), "nccl"),
    (3, GenSpec(30, 64, 0.08, "socp4", seed=32), dict(mu=0.7, max_iters=600, check_every=20), "nccl"),
    # the fused peer-memory step's ordering (partials -> barrier -> reduce+update+broadcast -> barrier)
    (2, GenSpec(40, 90, 0.06, "lp", seed=31), dict(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=4000), "p2p"),
    (3, GenSpec(30, 64, 0.08, "socp4", seed=32), dict(mu=0.7, max_iters=600, check_every=20), "p2p"),
    # the NVLS step (switch reduction + multicast store, device barrier) in the same driver
    (3, GenSpec(30, 64, 0.08, "socp4", seed=32), dict(mu=0.7, max_iters=600, check_every=20), "nvls"),
])
def test_sharded_matches_oracle(tmp_path, world, spec, cfg_kw, mode):
    out = str(tmp_path / "res.npz")
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, spec, cfg_kw, out, mode == "p2p", mode == "nvls"), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(out)
    p = generate(spec)
    cfg = SolverConfig(**cfg_kw)
    ox, olam, otrace, _ = oracle.solve(p, cfg)
    assert list(got["iters"]) == [r["iter"] for r in otrace]
    assert list(got["status"]) == [r["status"] for r in otrace]
    assert rel_err(got["x"], ox) <= 1e-8
    assert rel_err(got["lam"], olam) <= 1e-8
    np.testing.assert_allclose(got["pobj"], [r["pobj"] for r in otrace], rtol=1e-9, atol=1e-9)


def test_partition_balanced_and_cone_aligned():
    p = generate(GenSpec(100, 400, 0.05, "socp4", seed=1))
    rows, cols = partition(p, 4)
    assert rows[0] == 0 and rows[-1] == 100 and cols[0] == 0 and cols[-1] == 400
    assert all(c % 4 == 0 for c in cols)            # K4 blocks never split
    nnz = np.bincount(p.A.rows, minlength=100)
    per = [nnz[rows[r]:rows[r + 1]].sum() for r in range(4)]
    assert max(per) - min(per) <= nnz.max() + 1     # balanced to within one row


class NumpyColBackend:
    """Test-only restatement of one column-sharded rank (cf_plan_col_step / cf_apply_A /
    cf_plan_row_update / parts) on its column slice with all rows."""

    def __init__(self, lp):
        self.device = torch.device("cpu")
        a = lp.A
        order = np.lexsort((a.rows, a.cols))
        self.rows, self.cols, self.vals = a.rows[order], a.cols[order], a.vals[order]
        self.m, self.n = a.num_rows, a.num_cols
        self.b = np.asarray(lp.b, dtype=np.float64)
        self.c = np.asarray(lp.c, dtype=np.float64)
        self.dloc = np.bincount(self.rows, weights=self.vals * self.vals, minlength=self.m)
        self.lam, self.h = np.zeros(self.m), np.zeros(self.m)
        self.x, self.z, self.d = np.zeros(self.n), np.zeros(self.n), np.zeros(self.n)
        self.cnt = np.bincount(self.cols, minlength=self.n).astype(np.float64)   # all rows: true counts
        self.sizes = np.asarray(lp.cones.block_sizes, dtype=np.int64)
        self.ax_t = torch.zeros(self.m, dtype=torch.float64)

    def row_norms(self):
        return torch.tensor(self.dloc), torch.zeros(self.m, dtype=torch.float64)

    def set_row_norms(self, d, am):
        d = d.numpy()
        self.fu, self.db = 1.0 / (1.0 + d), d * self.b

    def col_step(self, mu):
        h = self.h_t.numpy()[:self.m] if getattr(self, "h_t", None) is not None else self.h
        ath = np.bincount(self.cols, weights=self.vals * h[self.rows], minlength=self.n)
        fv = 1.0 / (1.0 + self.cnt)
        dm = self.d / mu
        xp = fv * ((((self.cnt * self.x) + ath) + self.z + dm) - self.c / mu)
        w = xp - dm
        zp = project_cones_host(self.sizes, w)
        self.d = self.d + mu * (zp - xp)
        self.x, self.z = xp, zp

    def partial_Ax(self):
        self.ax_t.copy_(torch.tensor(np.bincount(self.rows, weights=self.vals * self.x[self.cols], minlength=self.m)))
        return self.ax_t

    def row_update(self, mu, report):
        ax = self.ax_t.numpy()
        r = self.fu * (self.db + ax)
        self.lam = self.lam + mu * (r - self.b)
        self.h = (self.b - r) - self.lam / mu
        self.ax = ax.copy()

    def row_parts(self):
        pr = self.ax - self.b
        return np.array([np.sum(pr * pr), np.max(np.abs(pr)), np.max(np.abs(self.ax)), np.sum(self.b * self.lam),
                         float(not np.isfinite(self.lam).all())])

    def col_parts(self):
        atl = np.bincount(self.cols, weights=self.vals * self.lam[self.rows], minlength=self.n)
        dual = atl + self.c
        stat = dual - self.d
        if atl.size == 0:
            return np.zeros(8)
        return np.array([np.sum(dual * dual), np.max(np.abs(dual)), np.sum(stat * stat), np.max(np.abs(stat)),
                         np.max(np.abs(atl)), np.sum(self.c * self.x), np.max(np.abs(self.x - self.z)),
                         float(not (np.isfinite(self.x).all() and np.isfinite(self.z).all()))])

    def x_slice(self):
        return torch.tensor(self.x)

    def lam_full(self):
        return torch.tensor(self.lam)

    # the sharded row update (run_col_sharded shard_rows): cf_apply_A_async into the padded
    # reduce-scatter input, cf_plan_row_update_range / _row_parts_range, cf_plan_bind_h
    def ax_into(self, out):
        out[:self.m] = torch.tensor(np.bincount(self.rows, weights=self.vals * self.x[self.cols], minlength=self.m))

    def bind_h(self, h):
        self.h_t = h

    def row_update_range(self, mu, report, r0, r1, ax_slice):
        ax = ax_slice.numpy()
        r = self.fu[r0:r1] * (self.db[r0:r1] + ax)
        self.lam[r0:r1] = self.lam[r0:r1] + mu * (r - self.b[r0:r1])
        self.h_t.numpy()[r0:r1] = (self.b[r0:r1] - r) - self.lam[r0:r1] / mu

    def row_parts_range(self, r0, r1, ax_slice):
        if r1 <= r0:
            return np.zeros(5)
        ax = ax_slice.numpy()
        pr = ax - self.b[r0:r1]
        return np.array([np.sum(pr * pr), np.max(np.abs(pr)), np.max(np.abs(ax)),
                         np.sum(self.b[r0:r1] * self.lam[r0:r1]), float(not np.isfinite(self.lam[r0:r1]).all())])

    def lam_range(self, r0, r1):
        return torch.tensor(self.lam[r0:r1])

    def set_lam(self, lam_full):
        self.lam = lam_full.numpy().copy()


def _col_worker(rank, world, port, spec, cfg_kw, out_path, shard_rows=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_05027_b200.sharded import solve_col_sharded

        p = generate(spec)
        res = solve_col_sharded(p, SolverConfig(**cfg_kw), backend_factory=NumpyColBackend, shard_rows=shard_rows)
        if rank == 0:
            np.savez(out_path, x=res.x, lam=res.lam, iters=np.array([r.iter for r in res.trace]),
                     status=np.array([r.status for r in res.trace]),
                     pobj=np.array([r.pobj for r in res.trace]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,spec,cfg_kw,shard_rows", [
    (2, GenSpec(40, 90, 0.06, "lp", seed=41), dict(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=4000), True),
    (3, GenSpec(31, 64, 0.08, "socp4", seed=42), dict(mu=0.7, max_iters=600, check_every=20), True),   # padded blocks
    (3, GenSpec(30, 64, 0.08, "socp4", seed=42), dict(mu=0.7, max_iters=600, check_every=20), False),
])
def test_column_sharded_matches_oracle(tmp_path, world, spec, cfg_kw, shard_rows):
    """Column sharding reaches the oracle's iterates: reduce-scatter of A x + each rank's block
    of rows + all-gather of h (shard_rows), or one all-reduce of A x + every row on every rank."""
    out = str(tmp_path / "res.npz")
    port = _free_port()
    mp.start_processes(_col_worker, args=(world, port, spec, cfg_kw, out, shard_rows), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out)
    p = generate(spec)
    cfg = SolverConfig(**cfg_kw)
    ox, olam, otrace, _ = oracle.solve(p, cfg)
    assert list(got["iters"]) == [r["iter"] for r in otrace]
    assert list(got["status"]) == [r["status"] for r in otrace]
    assert rel_err(got["x"], ox) <= 1e-8
    assert rel_err(got["lam"], olam) <= 1e-8
    np.testing.assert_allclose(got["pobj"], [r["pobj"] for r in otrace], rtol=1e-9, atol=1e-9)


def test_choose_sharding_by_exchange_volume():
    from paper_2203_05027_b200.sharded import choose_sharding, exchange_bytes

    # C5 (m=50M < n=100M): the all-reduce of A x moves half the bytes of rows' two n-vector exchanges
    assert exchange_bytes(50_000_000, 100_000_000, 8, "rows") == 2 * 8 * 100_000_000 * 7 // 8
    assert exchange_bytes(50_000_000, 100_000_000, 8, "cols") == 2 * 8 * 50_000_000 * 7 // 8
    assert choose_sharding(50_000_000, 100_000_000, 8) == "cols"
    assert choose_sharding(100, 40, 2) == "rows"
    assert choose_sharding(64, 64, 4) == "rows"      # tie -> rows
    assert choose_sharding(10, 1000, 1) == "rows"    # one rank: nothing is exchanged
    with pytest.raises(ValueError):
        exchange_bytes(1, 1, 2, "diagonal")


def _auto_worker(rank, world, port, spec, cfg_kw, out_path, factory_name):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_05027_b200.sharded import solve_distributed

        p = generate(spec)
        factory = {"rows": NumpyRankBackend, "cols": NumpyColBackend}[factory_name]
        res = solve_distributed(p, SolverConfig(**cfg_kw), mode="auto", backend_factory=factory)
        if rank == 0:
            np.savez(out_path, x=res.x, lam=res.lam, iters=np.array([r.iter for r in res.trace]),
                     status=np.array([r.status for r in res.trace]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("spec,expect", [
    (GenSpec(40, 90, 0.06, "lp", seed=51), "cols"),    # m < n
    (GenSpec(90, 60, 0.06, "lp", seed=52), "rows"),    # m > n
])
def test_solve_distributed_auto_matches_oracle(tmp_path, spec, expect):
    """mode="auto" picks the layout by shape and still reaches the oracle's iterates (gloo, world 2)."""
    from paper_2203_05027_b200.sharded import choose_sharding

    assert choose_sharding(spec.m, spec.n, 2) == expect
    cfg_kw = dict(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=3000)
    out = str(tmp_path / "res.npz")
    mp.start_processes(_auto_worker, args=(2, _free_port(), spec, cfg_kw, out, expect), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    p = generate(spec)
    ox, olam, otrace, _ = oracle.solve(p, SolverConfig(**cfg_kw))
    assert list(got["iters"]) == [r["iter"] for r in otrace]
    assert list(got["status"]) == [r["status"] for r in otrace]
    assert rel_err(got["x"], ox) <= 1e-8
    assert rel_err(got["lam"], olam) <= 1e-8
