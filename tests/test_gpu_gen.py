"""Device instance generators: recipe and host == device parity.

cfgen.generate_device (the C2/C3 bench instances) must return the arrays of
cfgen.generate_host bit for bit — that is what lets the CPU reference arm of bench.py
build the same instance without the GPU. Both generators are checked against the
reference recipe (generate.py:103-140): distinct positions, nonzero values,
b = A Proj_K(xdot) and c = Proj_K(sdot) - A^T lamdot in canonical order (the order
np.bincount sums in, uv.py:106-131). devgen.generate_device (torch Philox; the
robust-LS and sharded instances) gets the same recipe check.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from paper_2203_05027_b200 import cfgen  # noqa: E402
from paper_2203_05027_b200.instances import project_cones_host  # noqa: E402


def _bits(a):
    a = a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)
    return a.view(np.int64) if a.dtype == np.float64 else a


def _same(a, b):
    return np.array_equal(_bits(a), _bits(b))


@pytest.mark.parametrize("m,n,dens,kind,seed", [
    (1000, 2000, 0.01, "lp", 0),            # C1 shape
    (50_000, 100_000, 2e-4, "lp", 3),        # 1e6 nonzeros, C2 structure (20/row)
    (20_000, 40_000, 5e-4, "socp4", 1),      # C3 structure, K4 cones
    (30, 40, 0.6, "lp", 2),                  # dense: the key-sort branch
    (7, 8, 0.05, "socp4", 5),                # 3 nonzeros
])
def test_device_equals_host(m, n, dens, kind, seed):
    h = cfgen.generate_host(m, n, dens, kind, seed)
    d = cfgen.generate_device(m, n, dens, kind, seed)
    try:
        for name in ("rows", "cols", "vals", "b", "c"):
            assert _same(getattr(d, name), getattr(h, name)), name
        assert _same(d.x_feas, h.x_feas) and _same(d.lam_feas, h.lam_feas) and _same(d.slack_feas, h.slack_feas)
        assert cfgen.fingerprint(d.rows, d.cols, d.vals, d.b, d.c) == cfgen.fingerprint(h.rows, h.cols, h.vals,
                                                                                         h.b, h.c)
    finally:
        d.plan.close()


def _recipe(m, n, kind, rows, cols, vals, b, c, xdot, x_feas, lam, slack_raw, slack):
    rows, cols, vals, b, c = (a.detach().cpu().numpy() for a in (rows, cols, vals, b, c))
    x_feas, lam, slack = (a.detach().cpu().numpy() for a in (x_feas, lam, slack))
    o = vals.size
    key = cols * m + rows
    assert np.all(np.diff(key) > 0), "canonical order, distinct positions"
    assert rows.min() >= 0 and rows.max() < m and cols.min() >= 0 and cols.max() < n
    assert np.all(vals != 0.0) and np.all(np.isfinite(vals))
    assert abs(vals.mean()) < 5.0 / np.sqrt(o) + 1e-3 and abs(vals.std() - 1.0) < 0.01
    sizes = cfgen.cone_sizes(n, kind)
    if xdot is not None:
        assert _same(x_feas, project_cones_host(sizes, xdot))
        assert _same(slack, project_cones_host(sizes, slack_raw))
    # b = A Proj_K(xdot) and c = s - A^T lam, summed in canonical order (bit-for-bit)
    assert _same(b, np.bincount(rows, weights=vals * x_feas[cols], minlength=m))
    assert _same(c, slack - np.bincount(cols, weights=vals * lam[rows], minlength=n))


def test_cfgen_device_recipe_1e6():
    m, n, dens = 50_000, 100_000, 2e-4
    d = cfgen.generate_device(m, n, dens, "lp", 0)
    try:
        xdot = cfgen.normals(0, 2, 0, n)
        sraw = cfgen.normals(0, 4, 0, n)
        _recipe(m, n, "lp", d.rows, d.cols, d.vals, d.b, d.c, xdot, d.x_feas, d.lam_feas, sraw, d.slack_feas)
    finally:
        d.plan.close()


def test_devgen_philox_recipe_1e6():
    """devgen.generate_device (torch Philox stream): same recipe, b and c through the plan's
    operators. Re-derive the witness draws from the generator's seed."""
    from paper_2203_05027_b200 import devgen

    m, n, dens = 50_000, 100_000, 2e-4
    inst = devgen.generate_device(m, n, dens, "lp", seed=3)
    try:
        gen = torch.Generator(device="cuda")
        gen.manual_seed(3)
        # replay the stream: positions, values, then xdot, lam, sdot (devgen.py:126-165)
        o = inst.o
        devgen._distinct_positions(torch, gen, m * n, o, torch.device("cuda"))
        v = torch.randn(o, generator=gen, device="cuda", dtype=torch.float64)
        while bool((v == 0).any()):
            v[v == 0] = torch.randn(int((v == 0).sum()), generator=gen, device="cuda", dtype=torch.float64)
        xdot = torch.randn(n, generator=gen, device="cuda", dtype=torch.float64)
        lam = torch.randn(m, generator=gen, device="cuda", dtype=torch.float64)
        sd = torch.randn(n, generator=gen, device="cuda", dtype=torch.float64)
        xf = torch.clamp(xdot, min=0.0) + 0.0
        s = torch.clamp(sd, min=0.0) + 0.0
        order = torch.sort(inst.cols * m + inst.rows).indices
        r, cc, vv = inst.rows[order], inst.cols[order], inst.vals[order]
        _recipe(m, n, "lp", r, cc, vv, inst.b, inst.c, None, xf, lam, None, s)
    finally:
        inst.plan.close()
