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


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, spec, cfg_kw, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = generate(spec)
        cfg = SolverConfig(**cfg_kw)

        res = solve_sharded(p, cfg, backend_factory=NumpyRankBackend)
        if rank == 0:
            np.savez(out_path, x=res.x, lam=res.lam, iters=np.array([r.iter for r in res.trace]),
                     status=np.array([r.status for r in res.trace]),
                     pobj=np.array([r.pobj for r in res.trace]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,spec,cfg_kw", [
    (2, GenSpec(40, 90, 0.06, "lp", seed=31), dict(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=4000)),
    (3, GenSpec(30, 64, 0.08, "socp4", seed=32), dict(mu=0.7, max_iters=600, check_every=20)),
])
def test_sharded_matches_oracle(tmp_path, world, spec, cfg_kw):
    out = str(tmp_path / "res.npz")
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, spec, cfg_kw, out), nprocs=world, join=True, start_method="spawn")
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
        ath = np.bincount(self.cols, weights=self.vals * self.h[self.rows], minlength=self.n)
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


def _col_worker(rank, world, port, spec, cfg_kw, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2203_05027_b200.sharded import solve_col_sharded

        p = generate(spec)
        res = solve_col_sharded(p, SolverConfig(**cfg_kw), backend_factory=NumpyColBackend)
        if rank == 0:
            np.savez(out_path, x=res.x, lam=res.lam, iters=np.array([r.iter for r in res.trace]),
                     status=np.array([r.status for r in res.trace]),
                     pobj=np.array([r.pobj for r in res.trace]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,spec,cfg_kw", [
    (2, GenSpec(40, 90, 0.06, "lp", seed=41), dict(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4, max_iters=4000)),
    (3, GenSpec(30, 64, 0.08, "socp4", seed=42), dict(mu=0.7, max_iters=600, check_every=20)),
])
def test_column_sharded_matches_oracle(tmp_path, world, spec, cfg_kw):
    """Column sharding (one all-reduce of A x per iteration) reaches the oracle's iterates."""
    out = str(tmp_path / "res.npz")
    port = _free_port()
    mp.start_processes(_col_worker, args=(world, port, spec, cfg_kw, out), nprocs=world, join=True,
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
