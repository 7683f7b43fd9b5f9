"""Counter-based instance generator: the SAME arrays from numpy (host) and CUDA (device).

Bench tooling for the large configs (C2: 1e8 nonzeros, C3: 4e7). The recipe is the
reference generator's (generate.py:1-18, :82-140):

1. positions: the first ``count`` distinct cells of a uniform stream over the m*n grid
   (row-major cell index), sorted — ``_sample_positions`` (generate.py:82-100);
2. values: N(0,1), one per position in sorted position order (generate.py:112-117);
3. b = A Proj_K(xdot), xdot ~ N(0,1)^n (generate.py:124-126);
4. bounded mode: c = Proj_K(sdot) - A^T lamdot, lamdot ~ N(0,1)^m, sdot ~ N(0,1)^n
   (generate.py:128-132);

entries stored canonically (column-major, generate.py:119). Only the random stream
differs: numpy's PCG64 is a sequential stream, so instead every draw k of stream s is
``H(seed, s, k)`` (the splitmix64 finaliser over a Weyl sequence), a pure function of
its index, and normals come from Wichura's AS241 inverse CDF evaluated with a fixed
sequence of IEEE-rounded + - * / and sqrt plus a log built from the same operations
(frexp + atanh series). Every one of those operations rounds identically in numpy and
in CUDA (``csrc/cf_gen.cu`` uses __dadd_rn/__dmul_rn/__ddiv_rn/__dsqrt_rn, no FMA), and
the sums behind b and c run in canonical order (np.bincount here, the plan's
bit-identical segment sums on the device). So ``generate_host`` (numpy only, never
loads libcfb200 — the CPU reference arm of bench.py builds its instance with it) and
``generate_device`` return bit-identical arrays; tests/test_gpu_gen.py checks it, and
bench.py prints ``fingerprint()`` of the arrays on both arms.

Streams: 0 cell candidates, 1 values, 2 xdot, 3 lamdot, 4 sdot, 5 dense-case cell keys.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

__all__ = ["GEN_VERSION", "raw_u64", "normals", "distinct_cells", "HostInstance", "generate_host",
           "generate_device", "fingerprint", "cone_sizes"]

GEN_VERSION = 1

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_STREAM_MUL = np.uint64(0xD1B54A32D192ED03)
_CHUNK = 1 << 22


def _mix(z):
    """splitmix64 finaliser, in place on a uint64 array."""
    z ^= z >> np.uint64(30)
    z *= _M1
    z ^= z >> np.uint64(27)
    z *= _M2
    z ^= z >> np.uint64(31)
    return z


def _stream_base(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        z = np.array([(int(seed) ^ (int(stream) * int(_STREAM_MUL))) & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
        return _mix(z)[0]


def raw_u64(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """Draws start .. start+count-1 of stream ``stream``: mix(base + (k+1)*golden)."""
    base = _stream_base(seed, stream)
    with np.errstate(over="ignore"):
        k = np.arange(start + 1, start + 1 + count, dtype=np.uint64)
        k *= _GOLDEN
        k += base
        return _mix(k)


# ---------------------------------------------------------------- deterministic log and AS241
_SQRT_HALF = 0.7071067811865476
_LN2 = 0.6931471805599453
_LOG_SERIES = tuple(1.0 / (2 * k + 1) for k in range(13))   # atanh series: 1, 1/3, ..., 1/25

# Wichura, AS241 PPND16 (Applied Statistics 37, 1988): central region |q| <= 0.425
_A = (3.3871328727963666080e0, 1.3314166789178437745e+2, 1.9715909503065514427e+3, 1.3731693765509461125e+4,
      4.5921953931549871457e+4, 6.7265770927008700853e+4, 3.3430575583588128105e+4, 2.5090809287301226727e+3)
_B = (1.0, 4.2313330701600911252e+1, 6.8718700749205790830e+2, 5.3941960214247511077e+3,
      2.1213794301586595867e+4, 3.9307895800092710610e+4, 2.8729085735721942674e+4, 5.2264952788528545610e+3)
# r = sqrt(-log(min(p, 1-p))) <= 5
_C = (1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0, 3.64784832476320460504e0,
      1.27045825245236838258e0, 2.41780725177450611770e-1, 2.27238449892691845833e-2, 7.74545014278341407640e-4)
_D = (1.0, 2.05319162663775882187e0, 1.67638483018380384940e0, 6.89767334985100004550e-1,
      1.48103976427480074590e-1, 1.51986665636164571966e-2, 5.47593808499534494600e-4, 1.05075007164441684324e-9)
# r > 5
_E = (6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0, 2.96560571828504891230e-1,
      2.65321895265761230930e-2, 1.24266094738807843860e-3, 2.71155556874348757815e-5, 2.01033439929228813265e-7)
_F = (1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1, 1.48753612908506148525e-2,
      7.86869131145613259100e-4, 1.84631831751005468180e-5, 1.42151175831644588870e-7, 2.04426310338993978564e-15)


def _horner(coef, r):
    """((c7 r + c6) r + ...) r + c0 — one rounded multiply and one rounded add per step."""
    acc = np.full(r.shape, coef[7])
    for c in coef[6::-1]:
        acc *= r
        acc += c
    return acc


def _dlog(x):
    """log(x) for x > 0 from frexp and the atanh series: only rounded + - * /."""
    m, e = np.frexp(x)
    small = m < _SQRT_HALF
    m = np.where(small, m * 2.0, m)
    e = (e - small).astype(np.float64)
    f = m - 1.0
    s = f / (2.0 + f)
    z = s * s
    acc = np.full(z.shape, _LOG_SERIES[12])
    for c in _LOG_SERIES[11::-1]:
        acc *= z
        acc += c
    return e * _LN2 + (2.0 * s) * acc


def _normal_from_raw(r):
    """AS241 inverse normal CDF at p = ((r >> 12) + 0.5) / 2^52 (never 0, 1 or 0.5)."""
    p = ((r >> np.uint64(12)).astype(np.float64) + 0.5) * (1.0 / 4503599627370496.0)
    q = p - 0.5
    out = np.empty(p.shape)
    mid = np.abs(q) <= 0.425
    qm = q[mid]
    rr = 0.180625 - qm * qm
    out[mid] = qm * _horner(_A, rr) / _horner(_B, rr)
    tail = ~mid
    if tail.any():
        qt = q[tail]
        pt = p[tail]
        rt = np.where(qt < 0.0, pt, 1.0 - pt)
        rt = np.sqrt(-_dlog(rt))
        near = rt <= 5.0
        val = np.empty(rt.shape)
        r1 = rt[near] - 1.6
        val[near] = _horner(_C, r1) / _horner(_D, r1)
        r2 = rt[~near] - 5.0
        val[~near] = _horner(_E, r2) / _horner(_F, r2)
        out[tail] = np.where(qt < 0.0, -val, val)
    return out


def _threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def normals(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """N(0,1) draws start .. start+count-1 of stream ``stream`` (chunked over host threads)."""
    out = np.empty(count)

    def one(c0):
        c1 = min(count, c0 + _CHUNK)
        out[c0:c1] = _normal_from_raw(raw_u64(seed, stream, start + c0, c1 - c0))

    chunks = range(0, count, _CHUNK)
    if count > _CHUNK:
        with ThreadPoolExecutor(_threads()) as ex:
            list(ex.map(one, chunks))
    else:
        for c0 in chunks:
            one(c0)
    return out


def _cells_u64(seed: int, start: int, count: int, total: int) -> np.ndarray:
    out = np.empty(count, dtype=np.int64)
    tot = np.uint64(total)

    def one(c0):
        c1 = min(count, c0 + _CHUNK)
        out[c0:c1] = (raw_u64(seed, 0, start + c0, c1 - c0) % tot).astype(np.int64)

    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(one, range(0, count, _CHUNK)))
    return out


def distinct_cells(seed: int, total: int, count: int) -> np.ndarray:
    """The first ``count`` distinct values of the stream H(seed, 0, k) mod total, sorted.

    Same definition as generate.py:82-100 over this generator's stream. When the cells
    would be a large fraction of the grid (2*count >= total) the stream would mostly
    collide; then the cells are the ``count`` smallest keys (H(seed, 5, cell) >> 1, ties by
    cell), sorted — the analogue of the reference's permutation fallback."""
    if count > total:
        raise ValueError(f"cannot place {count} nonzeros in {total} cells")
    if count == 0:
        return np.zeros(0, dtype=np.int64)
    if 2 * count >= total:
        keys = (raw_u64(seed, 5, 0, total) >> np.uint64(1)).astype(np.int64)
        pick = np.argsort(keys, kind="stable")[:count]
        return np.sort(pick.astype(np.int64))
    L = count + count // 8 + 16
    while True:
        cand = _cells_u64(seed, 0, L, total)
        s = np.sort(cand)
        dup = s[1:] == s[:-1]
        first = np.ones(L, dtype=bool)
        if dup.any():
            dvals = np.unique(s[1:][dup])
            pos = np.searchsorted(dvals, cand)
            pos[pos == dvals.size] = 0
            hit = np.flatnonzero(dvals[pos] == cand)          # every occurrence of a repeated cell
            hv = cand[hit]
            order = np.lexsort((hit, hv))                       # by cell, then stream index
            hv, hit = hv[order], hit[order]
            later = np.concatenate(([False], hv[1:] == hv[:-1]))
            first[hit[later]] = False
        cum = np.cumsum(first)
        if cum[-1] >= count:
            T = int(np.searchsorted(cum, count)) + 1          # draws used: the count-th distinct is draw T-1
            uniq = s[np.concatenate(([True], ~dup))]
            drop = np.sort(cand[T:][first[T:]])                # distinct cells first drawn after T
            if drop.size:
                keep = np.ones(uniq.size, dtype=bool)
                keep[np.searchsorted(uniq, drop)] = False
                uniq = uniq[keep]
            assert uniq.size == count
            return uniq
        L = L + 2 * (count - int(cum[-1])) + 1024


# ---------------------------------------------------------------- instances
def cone_sizes(n: int, cone_kind: str) -> np.ndarray:
    if cone_kind == "lp":
        return np.ones(n, dtype=np.int64)
    if cone_kind == "socp4":
        if n % 4:
            raise ValueError("socp4 requires n divisible by 4")
        return np.full(n // 4, 4, dtype=np.int64)
    raise ValueError(f"cone_kind must be 'lp' or 'socp4', got {cone_kind!r}")


@dataclass
class HostInstance:
    m: int
    n: int
    o: int
    cone_kind: str
    rows: np.ndarray   # int64 [o], canonical (column-major, then row)
    cols: np.ndarray
    vals: np.ndarray   # float64 [o]
    b: np.ndarray
    c: np.ndarray
    block_sizes: np.ndarray
    x_feas: np.ndarray
    lam_feas: np.ndarray
    slack_feas: np.ndarray

    def problem(self):
        """This package's ProblemInstance (the reference's duck-typed layout)."""
        from .problem import ConeSpec, ProblemInstance, TripletMatrix

        return ProblemInstance(TripletMatrix(self.m, self.n, self.rows, self.cols, self.vals), self.b, self.c,
                               ConeSpec(self.block_sizes))


def _nnz(m: int, n: int, density: float) -> int:
    o = int(round(m * n * density))   # GenSpec.nnz (generate.py:60-62)
    if o < 1:
        raise ValueError(f"m*n*density rounds to {o} < 1 nonzero")
    return o


def _canonical_order(cols, n: int, o: int) -> np.ndarray:
    """Permutation from row-major to canonical (column-major, then row) order: a stable
    sort by column. Packs (column, position) into one int64 key when it fits, because
    numpy's unstable int64 sort is ~10x faster than its argsort (C2: 2 s vs 23 s)."""
    pbits = max(1, int(o - 1).bit_length())
    if int(n - 1).bit_length() + pbits <= 62:
        key = cols << np.int64(pbits)
        key |= np.arange(o, dtype=np.int64)
        key.sort()
        key &= np.int64((1 << pbits) - 1)
        return key
    return np.argsort(cols, kind="stable")


def generate_host(m: int, n: int, density: float, cone_kind: str = "lp", seed: int = 0) -> HostInstance:
    """The instance on the host, numpy only (no GPU, libcfb200 never loaded)."""
    from .instances import project_cones_host

    sizes = cone_sizes(n, cone_kind)
    o = _nnz(m, n, density)
    cells = distinct_cells(seed, m * n, o)
    rows, cols = cells // n, cells % n
    del cells
    vals = normals(seed, 1, 0, o)
    order = _canonical_order(cols, n, o)
    rows, cols, vals = rows[order], cols[order], vals[order]
    del order
    x_feas = project_cones_host(sizes, normals(seed, 2, 0, n))
    b = np.bincount(rows, weights=vals * x_feas[cols], minlength=m)          # U (V^T x), uv.py:106-131
    lam = normals(seed, 3, 0, m)
    slack = project_cones_host(sizes, normals(seed, 4, 0, n))
    c = slack - np.bincount(cols, weights=vals * lam[rows], minlength=n)    # s - V (U^T lam)
    return HostInstance(m, n, o, cone_kind, rows, cols, vals, b, c, sizes, x_feas, lam, slack)


def generate_device(m: int, n: int, density: float, cone_kind: str = "lp", seed: int = 0,
                    stream: int | None = None, keep_plan: bool = True):
    """The same instance built on the GPU (cf_gen_* kernels + torch sorts + the plan's operators).

    Returns a devgen.DeviceInstance whose plan is already built from the arrays."""
    import torch

    from ._lib import check, lib
    from .devgen import DeviceInstance
    from .engine import DevicePlan

    dev = torch.device("cuda")
    sizes = cone_sizes(n, cone_kind)
    o = _nnz(m, n, density)
    total = m * n
    cs = torch.cuda.current_stream().cuda_stream if stream is None else stream
    L = lib()

    def gen_cells(start, count, out):
        check(L.cf_gen_cells(seed, start, count, total, out.data_ptr(), cs), "cf_gen_cells")

    def gen_normals(s, count):
        out = torch.empty(count, dtype=torch.float64, device=dev)
        if count:
            check(L.cf_gen_normal(seed, s, 0, count, out.data_ptr(), cs), "cf_gen_normal")
        return out

    if 2 * o >= total:
        keys = torch.empty(total, dtype=torch.int64, device=dev)
        check(L.cf_gen_keys(seed, 5, 0, total, keys.data_ptr(), cs), "cf_gen_keys")
        pick = torch.sort(keys, stable=True).indices[:o]
        cells = torch.sort(pick).values
        del keys, pick
    else:
        Ld = o + o // 8 + 16
        while True:
            cand = torch.empty(Ld, dtype=torch.int64, device=dev)
            gen_cells(0, Ld, cand)
            s, perm = torch.sort(cand, stable=True)
            dup = s[1:] == s[:-1]
            first = torch.ones(Ld, dtype=torch.bool, device=dev)
            first[perm[1:][dup]] = False          # stable: later draws of a repeated cell
            cum = torch.cumsum(first, 0)
            got = int(cum[-1])
            if got >= o:
                T = int(torch.searchsorted(cum, torch.tensor([o], device=dev, dtype=cum.dtype))) + 1
                cells = torch.sort(cand[:T][first[:T]]).values
                del cand, s, perm, dup, first, cum
                break
            Ld = Ld + 2 * (o - got) + 1024
    rows = cells // n
    cols = cells % n
    del cells
    vals = gen_normals(1, o)
    order = torch.sort(cols * m + rows).indices
    rows, cols, vals = rows[order], cols[order], vals[order]
    del order
    b = torch.zeros(m, dtype=torch.float64, device=dev)
    c = torch.zeros(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    plan = DevicePlan.from_device(m, n, o, rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), b.data_ptr(),
                                  c.data_ptr(), sizes, stream=stream)
    xf = torch.empty(n, dtype=torch.float64, device=dev)
    xdot = gen_normals(2, n)
    torch.cuda.synchronize()
    plan.project(xdot.data_ptr(), xf.data_ptr())
    plan.apply_A(xf.data_ptr(), b.data_ptr())                 # b = A Proj_K(xdot)
    lam = gen_normals(3, m)
    sd = gen_normals(4, n)
    s_ = torch.empty_like(sd)
    torch.cuda.synchronize()
    plan.project(sd.data_ptr(), s_.data_ptr())
    atl = torch.empty(n, dtype=torch.float64, device=dev)
    plan.apply_At(lam.data_ptr(), atl.data_ptr())
    c.copy_(s_ - atl)                                          # c = Proj_K(sdot) - A^T lamdot
    torch.cuda.synchronize()
    plan.set_rhs(b.data_ptr(), c.data_ptr(), on_device=True)
    check(L.cf_plan_sync(plan.handle))
    inst = DeviceInstance(m, n, o, cone_kind, rows, cols, vals, b, c, sizes, plan if keep_plan else None)
    inst.x_feas, inst.lam_feas, inst.slack_feas = xf, lam, s_
    if not keep_plan:
        plan.close()
    return inst


def fingerprint(rows, cols, vals, b, c) -> str:
    """Order-sensitive 64-bit sums of the arrays' bit patterns (numpy or torch arrays): equal
    fingerprints on both bench arms mean the same instance. Wrapping int64 sums of
    (value * (index+1)) — identical in numpy and torch because integer addition is exact."""
    parts = []
    for a in (rows, cols, vals, b, c):
        if hasattr(a, "detach"):          # torch
            import torch

            v = a.contiguous().view(torch.int64) if a.dtype == torch.float64 else a.to(torch.int64)
            w = torch.arange(1, v.numel() + 1, device=v.device, dtype=torch.int64)
            s = int(((v * w) ^ (v >> 17)).sum().item())
        else:
            v = np.ascontiguousarray(a)
            v = v.view(np.int64) if v.dtype == np.float64 else v.astype(np.int64)
            with np.errstate(over="ignore"):
                w = np.arange(1, v.size + 1, dtype=np.int64)
                s = int(((v * w) ^ (v >> 17)).sum(dtype=np.int64))
        parts.append(f"{s & 0xFFFFFFFFFFFFFFFF:016x}")
    return "-".join(parts)
