"""Small solves that exercise every engine, for memory-safety checking.

    CF_LIB_PATH=paper_2203_05027_b200/libcfb200_checked.so python tools/sanitize_cases.py plan

compute-sanitizer is closed on the GPU pool, so the checked build (-DCF_CHECKED=1:
device bounds asserts that __trap() on any out-of-range index, guard canaries behind
every device buffer verified on release) stands in for memcheck; tests/test_gpu_checked.py
runs every case with it.

Each case drives one engine through the C ABI on a small instance and checks the
result against the oracle, so a sanitizer run also proves the path computed what it
should under instrumentation. Cases:
  plan        the k_pass chain (CF_NO_CLUSTER), direct engine, LP + K4 cones + mixed cones
  plan_knobs  the same with forced row panels / column bands / large tiles (carries, bands)
  cluster1/8/16  k_cluster at that cluster size (CF_CLUSTER_SIZE)
  batch       k_batch (solve_batch over 64 problems)
  gen         the cfgen device generator kernels
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _check(p, res, cfg):
    import oracle

    ox, olam, otrace, _ = oracle.solve(p, cfg)
    assert res.report.iter == otrace[-1]["iter"], (res.report.iter, otrace[-1]["iter"])
    err = np.max(np.abs(res.x - ox)) / (1 + np.max(np.abs(ox)))
    assert err < 1e-8, err


def main(case):
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve, solve_batch

    cfg = SolverConfig(eps_prim=1e-3, eps_dual=1e-3, eps_gap=1e-3, max_iters=400)
    if case in ("plan", "plan_knobs"):
        os.environ["CF_NO_CLUSTER"] = "1"
        if case == "plan_knobs":
            os.environ["CF_PANEL_MB"] = "0.002"
            os.environ["CF_BAND_MB"] = "0.0005"
            os.environ["CF_FORCE_LARGE_TILES"] = "1"
        for spec in (GenSpec(60, 150, 0.05, "lp", seed=1), GenSpec(40, 120, 0.06, "socp4", seed=2)):
            p = generate(spec)
            _check(p, solve(p, cfg), cfg)
        from paper_2203_05027_b200 import ConeSpec, ProblemInstance
        q = generate(GenSpec(50, 96, 0.08, "lp", seed=3))
        sizes = [3, 1, 1, 40, 5, 2, 1, 1, 4, 38]   # mixed cones incl. a 40-wide block
        mq = ProblemInstance(q.A, q.b, q.c, ConeSpec(tuple(sizes)))
        _check(mq, solve(mq, cfg), cfg)
    elif case.startswith("cluster"):
        os.environ["CF_CLUSTER_SIZE"] = case[len("cluster"):]
        from paper_2203_05027_b200 import api

        p = generate(GenSpec(300, 600, 0.03, "lp", seed=4))
        res = api._solve_cluster(p, cfg)   # direct: solve() skips the cluster path when CF_LIB_PATH is set
        assert res is not None and api._LAST_CLUSTER == int(case[len("cluster"):]), api._LAST_CLUSTER
        _check(p, res, cfg)
    elif case == "batch":
        probs = [generate(GenSpec(30, 60, 0.1, "lp", seed=s)) for s in range(64)]
        res = solve_batch(probs, cfg)
        for p, r in list(zip(probs, res))[:4]:
            _check(p, r, cfg)
    elif case == "gen":
        from paper_2203_05027_b200 import cfgen

        d = cfgen.generate_device(200, 400, 0.02, "socp4", 0)
        h = cfgen.generate_host(200, 400, 0.02, "socp4", 0)
        assert np.array_equal(d.b.cpu().numpy(), h.b)
        d.plan.close()
    else:
        raise SystemExit(f"unknown case {case}")
    from paper_2203_05027_b200 import _lib

    viol = int(_lib.lib().cf_debug_guard_violations())
    if viol > 0:
        raise SystemExit(f"case {case}: {viol} guard violation(s)")
    print(f"case {case}: ok (guard violations: {viol})")


if __name__ == "__main__":
    main(sys.argv[1])
