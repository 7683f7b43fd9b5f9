"""Per-pass timing of the plan loop (cf_plan_set_profiling): every iteration, or every k-th with
the sums scaled to the whole loop (the bench samples every 10th so the events do not break the
passes' programmatic-launch overlap)."""

import pytest

pytestmark = pytest.mark.gpu


def test_sampled_pass_timing_scales_to_the_loop():
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate
    from paper_2203_05027_b200.api import build_plan, norms
    from paper_2203_05027_b200.engine import config_struct

    p = generate(GenSpec(3000, 6000, 0.004, "lp", seed=4))
    cfg = SolverConfig(max_iters=400, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
    with build_plan(p) as plan:
        bn, cn = norms(p.b), norms(p.c)
        plan.set_state(1.0, None, export=False)
        plan.run(config_struct(cfg, bn, cn), want_x=False)   # warm-up: first-launch costs out of the way
        res = {}
        for stride in (1, 10, 0):
            plan.set_state(1.0, None, export=False)
            plan.set_profiling(stride > 0, stride=max(stride, 1))
            plan.run(config_struct(cfg, bn, cn), want_x=False)
            res[stride] = plan.last_timing()
        plan.set_profiling(False)
    for stride in (1, 10):
        t = res[stride]
        assert t["iters"] == 400
        assert t["row_pass_ms"] > 0 and t["col_pass_ms"] > 0
        assert t["row_pass_ms"] + t["col_pass_ms"] <= 2.0 * t["loop_ms"]
    # the sampled sums, scaled to 400 iterations, agree with the full sums to timing noise
    # (a ~10 us pass on a shared box: a wide band)
    for key in ("row_pass_ms", "col_pass_ms"):
        assert 0.25 < res[10][key] / res[1][key] < 4.0, (key, res)
    assert res[0]["row_pass_ms"] == 0.0 and res[0]["col_pass_ms"] == 0.0
