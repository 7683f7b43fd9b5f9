"""GPU instance generator for the large configs (C2: 100M nonzeros) — bench tooling.

Same recipe as the reference generator (generate.py:1-18, :103-140), built on
the device because the host recipe needs ~16 GB and ~4 minutes at 1e8
nonzeros: distinct uniform cell positions, N(0,1) values (zeros redrawn), a
primal witness x = Proj_K(N(0,1)) with b = A x, and in bounded mode
c = Proj_K(N(0,1)) - A^T N(0,1). The random stream is torch's Philox, not
numpy's PCG64, so instances are not bit-identical to ``instances.generate``
for the same seed; both solvers are always fed the SAME arrays.

Returns device tensors plus the DevicePlan already built from them (A x and
A^T y of the witness products run through libcfb200's own operators).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .engine import DevicePlan

__all__ = ["DeviceInstance", "generate_device", "generate_device_shard", "generate_device_colshard", "c2_spec",
           "c3_spec", "to_host_problem"]


@dataclass
class DeviceInstance:
    m: int
    n: int
    o: int
    cone_kind: str
    rows: "object"   # torch int64 [o], row-major sorted
    cols: "object"   # torch int64 [o]
    vals: "object"   # torch float64 [o]
    b: "object"      # torch float64 [m]
    c: "object"      # torch float64 [n]
    block_sizes: np.ndarray
    plan: DevicePlan | None = None


def c2_spec():
    """C2: LP m=5M, n=10M, 100M nonzeros (density 2e-6)."""
    return dict(m=5_000_000, n=10_000_000, density=2e-6, cone_kind="lp")


def c3_spec():
    """C3: SOCP m=2M, n=4M, 40M nonzeros, 1M K4 cones."""
    return dict(m=2_000_000, n=4_000_000, density=5e-6, cone_kind="socp4")


def _distinct_positions(torch, gen, total: int, count: int, device):
    """count distinct cells uniform over [0, total), sorted (uniform without replacement)."""
    draw = count + count // 64 + 1024
    pos = torch.unique(torch.randint(0, total, (draw,), generator=gen, device=device, dtype=torch.int64))
    while pos.numel() < count:
        more = torch.randint(0, total, (2 * (count - pos.numel()) + 1024,), generator=gen, device=device,
                             dtype=torch.int64)
        pos = torch.unique(torch.cat([pos, more]))
    if pos.numel() > count:
        keep = torch.randperm(pos.numel(), generator=gen, device=device)[:count]
        pos = torch.sort(pos[keep]).values
    return pos


def rls_arrays(torch, gen, m: int, n: int, density: float, device):
    """Robust least squares in SOC form (the secondary mixed-cone instance).

    min sum_i t_i + 0.01 * 1^T (x+ + x-)   s.t.   u_i - F_i (x+ - x-) = -g_i,
    (t_i, u_i) in K4 (i < K), x+, x- >= 0 (p each).

    m = 3K rows (row 3i+r is component r of u_i); n = 4K + 2p columns: cone i owns
    [4i, 4i+4), then x+ and x-. Each row holds u's 1.0 plus k F entries, each stored
    twice (+f on x+, -f on x-), so density*n = 1 + 2k. The k columns of a row are
    h, h+s, ..., h+(k-1)s mod p with s < p/k, hence distinct. The t columns have no
    entries. Returns (rows, cols, vals, b, c, block_sizes) on `device`."""
    K = m // 3
    p2 = n - 4 * K
    if m != 3 * K or K < 1 or p2 < 2 or p2 % 2:
        raise ValueError("rls needs m = 3K and n = 4K + 2p, p >= 1")
    p = p2 // 2
    k = int(min(max(1, round((density * n - 1.0) / 2.0)), p))
    r = torch.arange(m, device=device, dtype=torch.int64)
    h = torch.randint(0, p, (m, 1), generator=gen, device=device, dtype=torch.int64)
    s = torch.randint(1, max(2, p // k + 1), (m, 1), generator=gen, device=device, dtype=torch.int64)
    j = (h + s * torch.arange(k, device=device, dtype=torch.int64)) % p            # [m, k] distinct per row
    f = torch.randn(m, k, generator=gen, device=device, dtype=torch.float64)
    while True:
        zero = f == 0.0
        nz = int(zero.sum())
        if nz == 0:
            break
        f[zero] = torch.randn(nz, generator=gen, device=device, dtype=torch.float64)
    u_col = 4 * (r // 3) + 1 + r % 3
    rows = torch.cat([r, r.repeat_interleave(k), r.repeat_interleave(k)])
    cols = torch.cat([u_col, (4 * K + j).reshape(-1), (4 * K + p + j).reshape(-1)])
    vals = torch.cat([torch.ones(m, device=device, dtype=torch.float64), f.reshape(-1), -f.reshape(-1)])
    b = -torch.randn(m, generator=gen, device=device, dtype=torch.float64)
    c = torch.zeros(n, device=device, dtype=torch.float64)
    c[0:4 * K:4] = 1.0
    c[4 * K:] = 0.01
    sizes = np.concatenate([np.full(K, 4, dtype=np.int64), np.ones(2 * p, dtype=np.int64)])
    return rows, cols, vals, b, c, sizes


def generate_device(m: int, n: int, density: float, cone_kind: str = "lp", seed: int = 0,
                    bounded_mode: bool = True, keep_plan: bool = True, stream: int | None = None) -> DeviceInstance:
    import torch

    dev = torch.device("cuda")
    if cone_kind == "rls":
        gen = torch.Generator(device=dev)
        gen.manual_seed(int(seed))
        rows, cols, vals, b, c, sizes = rls_arrays(torch, gen, m, n, density, dev)
        o = int(vals.numel())
        torch.cuda.synchronize()
        plan = DevicePlan.from_device(m, n, o, rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), b.data_ptr(),
                                      c.data_ptr(), sizes, stream=stream)
        inst = DeviceInstance(m, n, o, cone_kind, rows, cols, vals, b, c, sizes, plan if keep_plan else None)
        if not keep_plan:
            plan.close()
        return inst
    o = int(round(m * n * density))
    if o < 1:
        raise ValueError("instance has no nonzeros")
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(seed))
    pos = _distinct_positions(torch, gen, m * n, o, dev)
    rows = pos // n
    cols = pos % n
    del pos
    vals = torch.randn(o, generator=gen, device=dev, dtype=torch.float64)
    while True:
        zero = vals == 0.0
        nz = int(zero.sum())
        if nz == 0:
            break
        vals[zero] = torch.randn(nz, generator=gen, device=dev, dtype=torch.float64)
    if cone_kind == "lp":
        sizes = np.ones(n, dtype=np.int64)
    elif cone_kind == "socp4":
        if n % 4:
            raise ValueError("socp4 requires n divisible by 4")
        sizes = np.full(n // 4, 4, dtype=np.int64)
    else:
        raise ValueError(cone_kind)
    b = torch.zeros(m, dtype=torch.float64, device=dev)
    c = torch.zeros(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    plan = DevicePlan.from_device(m, n, o, rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), b.data_ptr(),
                                  c.data_ptr(), sizes, stream=stream)
    xdot = torch.randn(n, generator=gen, device=dev, dtype=torch.float64)
    xf = torch.empty_like(xdot)
    plan.project(xdot.data_ptr(), xf.data_ptr())
    plan.apply_A(xf.data_ptr(), b.data_ptr())                 # b = A Proj_K(xdot)
    if bounded_mode:
        lam = torch.randn(m, generator=gen, device=dev, dtype=torch.float64)
        sd = torch.randn(n, generator=gen, device=dev, dtype=torch.float64)
        s = torch.empty_like(sd)
        plan.project(sd.data_ptr(), s.data_ptr())
        atl = torch.empty(n, dtype=torch.float64, device=dev)
        plan.apply_At(lam.data_ptr(), atl.data_ptr())
        c.copy_(s - atl)                                       # c = Proj_K(s) - A^T lam
    else:
        c.copy_(torch.randn(n, generator=gen, device=dev, dtype=torch.float64))
    torch.cuda.synchronize()
    plan.set_rhs(b.data_ptr(), c.data_ptr(), on_device=True)
    inst = DeviceInstance(m, n, o, cone_kind, rows, cols, vals, b, c, sizes, plan if keep_plan else None)
    if not keep_plan:
        plan.close()
    return inst


def to_host_problem(inst: DeviceInstance):
    """Copy a device instance to a host ProblemInstance (this package's types)."""
    from .problem import ConeSpec, ProblemInstance, TripletMatrix

    a = TripletMatrix(inst.m, inst.n, inst.rows.cpu().numpy(), inst.cols.cpu().numpy(), inst.vals.cpu().numpy())
    return ProblemInstance(a, inst.b.cpu().numpy(), inst.c.cpu().numpy(), ConeSpec(inst.block_sizes))


def generate_device_shard(m: int, n: int, density: float, cone_kind: str, seed: int, rank: int, world: int,
                          group=None, stream: int | None = None):
    """Rank ``rank``'s row block of a row-sharded instance (C5), built on its GPU only.

    Rows [m*rank/world, m*(rank+1)/world) get their share of the nonzeros
    (uniform positions, N(0,1) values); the primal witness x and the dual slack
    draw are shared (same seed on every rank) so b_local = A_local Proj_K(x) and
    c = Proj_K(s) - sum_r A_r^T lam_r (an all-reduce) reproduce the generator
    recipe of generate.py:103-140 for the whole matrix. Returns
    (plan, row_cuts, col_cuts, c_slice tensor, b_norms, c_norms)."""
    import math

    import torch
    import torch.distributed as dist

    dev = torch.device("cuda")
    r0, r1 = m * rank // world, m * (rank + 1) // world
    ml = r1 - r0
    o = int(round(ml * n * density))
    g_local = torch.Generator(device=dev)
    g_local.manual_seed(int(seed) * 1000003 + rank)
    g_shared = torch.Generator(device=dev)
    g_shared.manual_seed(int(seed))
    pos = _distinct_positions(torch, g_local, ml * n, o, dev)
    rows, cols = pos // n, pos % n
    del pos
    vals = torch.randn(o, generator=g_local, device=dev, dtype=torch.float64)
    while True:   # zeros are redrawn (generate.py:112-117)
        zero = vals == 0.0
        nz = int(zero.sum())
        if nz == 0:
            break
        vals[zero] = torch.randn(nz, generator=g_local, device=dev, dtype=torch.float64)
    if cone_kind == "lp":
        sizes = np.ones(n, dtype=np.int64)
        unit = 1
    else:
        sizes = np.full(n // 4, 4, dtype=np.int64)
        unit = 4
    b = torch.zeros(ml, dtype=torch.float64, device=dev)
    c = torch.zeros(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    # the local plan's own column pass is never used (the driver updates column slices), so the
    # orthant is enough here; the cones enter through the slice update
    plan = DevicePlan.from_device(ml, n, o, rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), b.data_ptr(),
                                  c.data_ptr(), np.ones(n, dtype=np.int64), stream=stream)
    del rows, cols, vals
    xdot = torch.randn(n, generator=g_shared, device=dev, dtype=torch.float64)
    xf = _project(torch, xdot, unit)
    plan.apply_A(xf.data_ptr(), b.data_ptr())
    lam = torch.randn(ml, generator=g_local, device=dev, dtype=torch.float64)
    atl = torch.empty(n, dtype=torch.float64, device=dev)
    plan.apply_At(lam.data_ptr(), atl.data_ptr())
    dist.all_reduce(atl, op=dist.ReduceOp.SUM, group=group)
    s = _project(torch, torch.randn(n, generator=g_shared, device=dev, dtype=torch.float64), unit)
    c.copy_(s - atl)
    torch.cuda.synchronize()
    plan.set_rhs(b.data_ptr(), c.data_ptr(), on_device=True)
    row_cuts = [m * r // world for r in range(world + 1)]
    step = -(-n // world)
    step = -(-step // unit) * unit
    col_cuts = [min(n, r * step) for r in range(world)] + [n]
    lo, hi = col_cuts[rank], col_cuts[rank + 1]
    # global norms of b (distributed) and c (replicated): ||.||_inf and ||.||_2 as solver.py:200-203
    bb = torch.stack([b.abs().max() if ml else torch.zeros((), device=dev, dtype=torch.float64), (b * b).sum()])
    dist.all_reduce(bb[:1], op=dist.ReduceOp.MAX, group=group)
    sq = bb[1:].clone()
    dist.all_reduce(sq, op=dist.ReduceOp.SUM, group=group)
    b_norms = (float(bb[0]), math.sqrt(float(sq)))
    c_norms = (float(c.abs().max()), math.sqrt(float((c * c).sum())))
    cone_slice = None if unit == 1 else (np.arange(lo, hi + 1, 4) - lo).astype(np.int32)
    return plan, row_cuts, col_cuts, c[lo:hi].clone(), b_norms, c_norms, cone_slice


def generate_device_colshard(m: int, n: int, density: float, cone_kind: str, seed: int, rank: int, world: int,
                             group=None, stream: int | None = None):
    """Rank ``rank``'s column slice of a column-sharded instance (all rows), built on its GPU.

    Columns [c0, c1) (cone-aligned) get their share of the nonzeros; the primal witness and
    the dual draw are shared (same seed on every rank), so b = sum_r A_r Proj_K(x)_r (an
    all-reduce) and c_r = Proj_K(s)_r - A_r^T lam reproduce the generator recipe of
    generate.py:103-140 for the whole matrix. Returns (plan, col_cuts, b_norms, c_norms)."""
    import math

    import torch
    import torch.distributed as dist

    dev = torch.device("cuda")
    unit = 1 if cone_kind == "lp" else 4
    step = -(-n // world)
    step = -(-step // unit) * unit
    col_cuts = [min(n, r * step) for r in range(world)] + [n]
    c0, c1 = col_cuts[rank], col_cuts[rank + 1]
    nl = c1 - c0
    o = int(round(m * nl * density))
    g_local = torch.Generator(device=dev)
    g_local.manual_seed(int(seed) * 1000003 + rank)
    g_shared = torch.Generator(device=dev)
    g_shared.manual_seed(int(seed))
    pos = _distinct_positions(torch, g_local, m * nl, o, dev)
    rows, cols = pos // nl, pos % nl
    del pos
    vals = torch.randn(o, generator=g_local, device=dev, dtype=torch.float64)
    while True:   # zeros are redrawn (generate.py:112-117)
        zero = vals == 0.0
        nz = int(zero.sum())
        if nz == 0:
            break
        vals[zero] = torch.randn(nz, generator=g_local, device=dev, dtype=torch.float64)
    sizes = np.full(nl // unit, unit, dtype=np.int64)
    b = torch.zeros(m, dtype=torch.float64, device=dev)
    c = torch.zeros(nl, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    plan = DevicePlan.from_device(m, nl, o, rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), b.data_ptr(),
                                  c.data_ptr(), sizes, stream=stream)
    del rows, cols, vals
    xf = _project(torch, torch.randn(n, generator=g_shared, device=dev, dtype=torch.float64), unit)[c0:c1]
    xf = xf.contiguous()
    plan.apply_A(xf.data_ptr(), b.data_ptr())
    dist.all_reduce(b, op=dist.ReduceOp.SUM, group=group)
    lam = torch.randn(m, generator=g_shared, device=dev, dtype=torch.float64)
    atl = torch.empty(nl, dtype=torch.float64, device=dev)
    plan.apply_At(lam.data_ptr(), atl.data_ptr())
    s = _project(torch, torch.randn(n, generator=g_shared, device=dev, dtype=torch.float64), unit)[c0:c1]
    c.copy_(s - atl)
    torch.cuda.synchronize()
    plan.set_rhs(b.data_ptr(), c.data_ptr(), on_device=True)
    b_norms = (float(b.abs().max()), math.sqrt(float((b * b).sum())))
    cc = torch.stack([c.abs().max() if nl else torch.zeros((), device=dev, dtype=torch.float64), (c * c).sum()])
    mx = cc[:1].clone()
    sq = cc[1:].clone()
    dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
    dist.all_reduce(sq, op=dist.ReduceOp.SUM, group=group)
    c_norms = (float(mx), math.sqrt(float(sq)))
    return plan, col_cuts, b_norms, c_norms


def _project(torch, w, unit):
    if unit == 1:
        return torch.clamp(w, min=0.0) + 0.0
    v = w.view(-1, unit)
    head, tail = v[:, 0], v[:, 1:]
    alpha = torch.sqrt((tail * tail).sum(1))
    out = torch.zeros_like(v)
    keep = alpha <= head
    scale = ~(alpha <= -head) & ~keep
    out[keep] = v[keep]
    f = head[scale] / (2.0 * alpha[scale])
    out[scale, 1:] = 0.5 * tail[scale] + f[:, None] * tail[scale]
    out[scale, 0] = 0.5 * head[scale] + 0.5 * alpha[scale]
    return out.view(-1)
