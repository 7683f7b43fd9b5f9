"""Time-to-tolerance fixtures at the BASELINE structures, produced by the UNMODIFIED reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_headline_golden.py

Instances come from cfgen.generate_host (numpy; the same arrays cfgen.generate_device
builds on the GPU, tests/test_gpu_gen.py), so the GPU test regenerates them on the
device and compares its solve with what conefree.solve (solver.py:275-334) did here:
  c2s_1e5   C2 structure (20 nonzeros per row, 10 per column), m=5,000 n=10,000, o=1e5, LP
  c3s_20    C3 at 1/20 scale (same nonzeros per row/column), m=100,000 n=200,000, o=2e6,
            50,000 K4 cones
Both solved with SolverConfig(eps_prim=eps_dual=eps_gap=1e-4) (scs mode), cold start.
Stored: every report of the trace (13 fields + status), and x / lam (in full for c2s,
a fixed subsample of 4,096 entries each for c3s, plus their 2-norms).
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2203_05027_b200 import cfgen  # noqa: E402

CASES = {
    "c2s_1e5": dict(m=5_000, n=10_000, density=2e-3, kind="lp", full=True),
    "c3s_20": dict(m=100_000, n=200_000, density=1e-4, kind="socp4", full=False),
}
FIELDS = ("iter", "prim_res_inf", "prim_res_2", "dual_res_inf", "dual_res_2", "stat_res_inf", "stat_res_2",
          "ax_inf", "atl_inf", "cone_gap", "pobj", "dobj", "gap")


def main(names):
    from conefree.model import ConeSpec, ProblemInstance, TripletMatrix
    from conefree.solver import SolverConfig, solve

    for name in names:
        c = CASES[name]
        h = cfgen.generate_host(c["m"], c["n"], c["density"], c["kind"], 0)
        p = ProblemInstance(TripletMatrix(h.m, h.n, h.rows, h.cols, h.vals), h.b, h.c,
                            ConeSpec(tuple(int(s) for s in h.block_sizes)))
        t0 = time.perf_counter()
        res = solve(p, SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4))
        secs = time.perf_counter() - t0
        trace = np.array([[getattr(r, f) for f in FIELDS] for r in res.trace], dtype=np.float64)
        status = np.array([r.status for r in res.trace])
        out = dict(m=h.m, n=h.n, o=h.o, density=c["density"], kind=c["kind"], trace=trace, status=status,
                   fingerprint=cfgen.fingerprint(h.rows, h.cols, h.vals, h.b, h.c),
                   x_norm=np.linalg.norm(res.x), lam_norm=np.linalg.norm(res.lam), seconds=secs)
        if c["full"]:
            out.update(x=res.x, lam=res.lam)
        else:
            xi = np.linspace(0, h.n - 1, 4096).astype(np.int64)
            li = np.linspace(0, h.m - 1, 4096).astype(np.int64)
            out.update(x_idx=xi, x_sub=res.x[xi], lam_idx=li, lam_sub=res.lam[li])
        np.savez_compressed(os.path.join(HERE, f"headline_{name}.npz"), **out)
        print(name, res.report.iter, res.report.status, f"{secs:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(CASES))
