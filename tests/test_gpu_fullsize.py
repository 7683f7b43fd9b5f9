"""Full-size (BASELINE configs C2 and C3) checks through size-independent properties.

The oracle cannot iterate 1e8 nonzeros in test time, so at these sizes the device path is
checked against facts that hold at any size:
* the device compute_report (solver.py:206-242) equals a recomputation of the same residuals
  and objectives from the exported iterates with torch fp64 (A x and A^T lam by index_add_,
  a different summation order, hence a tolerance);
* cone_gap = max|x - z| has no summation: exact;
* z lies in the cone (Proj_K output, cones.py:78-91);
* two cold-start runs of the same plan give bit-identical iterates (SPEC determinism).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# relative tolerance for sums taken in another order over ~1e8 fp64 products
RTOL = 1e-9


def _close(got, want, scale):
    assert abs(got - want) <= RTOL * max(abs(want), scale), (got, want, scale)


@pytest.mark.parametrize("which", ["c2", "c3"])
def test_full_size_report_and_cone_properties(which):
    import torch

    from paper_2203_05027_b200 import cfgen
    from paper_2203_05027_b200.devgen import c2_spec, c3_spec

    spec = c2_spec() if which == "c2" else c3_spec()
    inst = cfgen.generate_device(spec["m"], spec["n"], spec["density"], spec["cone_kind"], 0)   # the bench instance
    plan = inst.plan
    try:
        plan.set_state(1.0, None, export=False)
        plan.iterate(1.0, 50)
        rep = plan.report(1.0)
        st = plan.get_state(want_yg=False)
        assert st["iter"] == 50 and rep["status"] == "running"

        dev = inst.vals.device
        x, z, dl, lam = (torch.from_numpy(st[k]).to(dev) for k in ("x", "z", "delta", "lam"))
        rows, cols, vals, b, c = inst.rows, inst.cols, inst.vals, inst.b, inst.c
        ax = torch.zeros(inst.m, dtype=torch.float64, device=dev).index_add_(0, rows, vals * x[cols])
        atl = torch.zeros(inst.n, dtype=torch.float64, device=dev).index_add_(0, cols, vals * lam[rows])
        prim, dual = ax - b, atl + c
        stat = dual - dl

        def norms(v):
            return float(v.abs().max()), float(torch.sqrt(torch.dot(v, v)))

        ax_inf, atl_inf = norms(ax)[0], norms(atl)[0]
        b_inf, c_inf = norms(b)[0], norms(c)[0]
        for key, v, scale in (("prim", prim, ax_inf + b_inf), ("dual", dual, atl_inf + c_inf),
                              ("stat", stat, atl_inf + c_inf + norms(dl)[0])):
            inf, two = norms(v)
            _close(rep[f"{key}_res_inf"], inf, scale)
            _close(rep[f"{key}_res_2"], two, scale)
        _close(rep["ax_inf"], ax_inf, ax_inf)
        _close(rep["atl_inf"], atl_inf, atl_inf)
        pobj, blam = float(torch.dot(c, x)), float(torch.dot(b, lam))
        obj_scale = float(torch.dot(c.abs(), x.abs()) + torch.dot(b.abs(), lam.abs()))
        _close(rep["pobj"], pobj, obj_scale)
        _close(rep["dobj"], -blam, obj_scale)
        _close(rep["gap"], pobj + blam, obj_scale)
        assert rep["cone_gap"] == float((x - z).abs().max())   # no summation: exact

        # z in K
        if spec["cone_kind"] == "lp":
            assert bool((z >= 0).all())
        else:
            # head >= |tail| up to rounding. The projection's tail 0.5w + (w0/(2 alpha))w
            # (cones.py:88-91) cancels when w0 ~ -alpha, so the rounding is relative to the
            # block's input scale, not to the (tiny) output: measured worst 1 ulp of |w|
            blk = z.view(-1, 4)
            tail = torch.sqrt((blk[:, 1:] ** 2).sum(1))
            scale = tail + blk[:, 0].abs() + x.view(-1, 4).abs().amax(1) + dl.view(-1, 4).abs().amax(1)
            assert bool((tail - blk[:, 0] <= 1e-12 * scale).all())

        # determinism: a second cold start of the same plan repeats the run bit for bit
        plan.set_state(1.0, None, export=False)
        plan.iterate(1.0, 50)
        st2 = plan.get_state(want_yg=False)
        for k in ("x", "z", "delta", "lam"):
            assert np.array_equal(st[k], st2[k]), k
    finally:
        plan.close()
        torch.cuda.synchronize()
