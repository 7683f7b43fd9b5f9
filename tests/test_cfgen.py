"""The counter-based instance generator's host half (cfgen.py), CPU only.

The device half and host == device are in tests/test_gpu_gen.py. Here: the stream and
the first-distinct rule against a literal pure-Python restatement, the AS241 normals
against scipy's ndtri, and the recipe of generate.py:103-140 on the host arrays.
"""

import numpy as np
import pytest

from paper_2203_05027_b200 import cfgen
from paper_2203_05027_b200.instances import project_cones_host

MASK = (1 << 64) - 1


def _mix_py(z):
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def _draw_py(seed, stream, k):
    base = _mix_py((seed ^ (stream * 0xD1B54A32D192ED03)) & MASK)
    return _mix_py((base + (k + 1) * 0x9E3779B97F4A7C15) & MASK)


def test_stream_matches_literal_splitmix():
    got = cfgen.raw_u64(7, 3, 1000, 50)
    want = [_draw_py(7, 3, 1000 + i) for i in range(50)]
    assert [int(v) for v in got] == want


def test_first_distinct_rule_matches_python_loop():
    """generate.py:82-100 semantics: the first `count` distinct cells of the stream, sorted."""
    for seed, total, count in ((0, 97, 40), (3, 1000, 300), (5, 50_000, 20_000), (9, 10, 10), (2, 400, 150)):
        got = cfgen.distinct_cells(seed, total, count)
        if 2 * count >= total:   # dense: the count smallest keys (H >> 1, ties by cell)
            keys = [(_draw_py(seed, 5, c) >> 1, c) for c in range(total)]
            want = sorted(c for _, c in sorted(keys)[:count])
        else:
            seen, order, k = set(), [], 0
            while len(order) < count:
                v = _draw_py(seed, 0, k) % total
                k += 1
                if v not in seen:
                    seen.add(v)
                    order.append(v)
            want = sorted(order)
        assert got.tolist() == want, (seed, total, count)


def test_normals_against_ndtri_and_moments():
    sp = pytest.importorskip("scipy.special")
    r = cfgen.raw_u64(0, 1, 0, 400_000)
    p = ((r >> np.uint64(12)).astype(np.float64) + 0.5) / 4503599627370496.0
    z = cfgen.normals(0, 1, 0, 400_000)
    ref = sp.ndtri(p)
    assert np.max(np.abs(z - ref) / np.maximum(1.0, np.abs(ref))) < 1e-14
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
    assert np.all(z != 0.0)
    # extreme p: both tail branches (r <= 5 and r > 5)
    far = np.array([1, 2, 2**20, 2**51 - 7, 2**52 - 1], dtype=np.uint64) << np.uint64(12)
    pf = ((far >> np.uint64(12)).astype(np.float64) + 0.5) / 4503599627370496.0
    assert np.allclose(cfgen._normal_from_raw(far), sp.ndtri(pf), rtol=1e-14, atol=0)


def test_chunked_normals_equal_one_shot():
    a = cfgen.normals(4, 2, 0, (1 << 22) + 1000)   # crosses a chunk boundary, threaded
    b = np.concatenate([cfgen.normals(4, 2, 0, 1 << 22), cfgen.normals(4, 2, 1 << 22, 1000)])
    assert np.array_equal(a.view(np.int64), b.view(np.int64))


@pytest.mark.parametrize("kind", ["lp", "socp4"])
def test_host_instance_recipe(kind):
    """generate.py:103-140 on the host arrays: distinct positions, nonzero N(0,1) values in
    position order, canonical order, b = A Proj_K(xdot), c = Proj_K(sdot) - A^T lamdot."""
    m, n, dens, seed = 300, 800, 0.02, 11
    h = cfgen.generate_host(m, n, dens, kind, seed)
    o = int(round(m * n * dens))
    assert h.o == o and h.rows.size == o
    key = h.cols * m + h.rows
    assert np.all(np.diff(key) > 0)                                  # canonical, distinct
    cells = np.sort(h.rows * n + h.cols)
    assert np.array_equal(cells, cfgen.distinct_cells(seed, m * n, o))
    # values in row-major position order
    rm = np.lexsort((h.cols, h.rows))
    assert np.array_equal(h.vals[rm].view(np.int64), cfgen.normals(seed, 1, 0, o).view(np.int64))
    assert np.all(h.vals != 0.0)
    sizes = cfgen.cone_sizes(n, kind)
    xf = project_cones_host(sizes, cfgen.normals(seed, 2, 0, n))
    assert np.array_equal(h.x_feas, xf)
    b = np.bincount(h.rows, weights=h.vals * xf[h.cols], minlength=m)
    assert np.array_equal(h.b.view(np.int64), b.view(np.int64))
    lam = cfgen.normals(seed, 3, 0, m)
    s = project_cones_host(sizes, cfgen.normals(seed, 4, 0, n))
    c = s - np.bincount(h.cols, weights=h.vals * lam[h.rows], minlength=n)
    assert np.array_equal(h.c.view(np.int64), c.view(np.int64))
    # A x_feas = b to rounding and the dual witness: A^T lam + c = s in K
    assert np.allclose(np.bincount(h.rows, weights=h.vals * h.x_feas[h.cols], minlength=m), h.b)
    if kind == "socp4":
        v = s.reshape(-1, 4)
        assert np.all(v[:, 0] >= np.sqrt((v[:, 1:] ** 2).sum(1)) - 1e-12)


def test_host_generator_deterministic_and_fingerprint():
    a = cfgen.generate_host(200, 500, 0.03, "lp", 5)
    b = cfgen.generate_host(200, 500, 0.03, "lp", 5)
    fa = cfgen.fingerprint(a.rows, a.cols, a.vals, a.b, a.c)
    assert fa == cfgen.fingerprint(b.rows, b.cols, b.vals, b.b, b.c)
    c = cfgen.generate_host(200, 500, 0.03, "lp", 6)
    assert fa != cfgen.fingerprint(c.rows, c.cols, c.vals, c.b, c.c)


def test_canonical_order_paths_agree():
    rng = np.random.default_rng(0)
    cols = np.sort(rng.integers(0, 1000, 5000))
    cols = rng.permutation(cols)
    packed = cfgen._canonical_order(cols, 1000, cols.size)
    assert np.array_equal(packed, np.argsort(cols, kind="stable"))
