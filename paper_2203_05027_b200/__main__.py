"""``python -m paper_2203_05027_b200 bench`` — the GPU bench sweep hook.

Runs ``benchrun.run_bench`` over a grid of generated instances and writes the
reference's bench CSV (``BENCH_COLUMNS``) plus the it/s, GB/s and roofline
columns. The reference's full command line (solve/generate, cli.py) is out of
scope; this is only the device bench entry point.
"""

from __future__ import annotations

import argparse
import sys


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2203_05027_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--nnz", required=True, help="target nonzero counts, comma separated")
    b.add_argument("--density", required=True, help="densities, comma separated")
    b.add_argument("--cone", default="lp", choices=("lp", "socp4"))
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--eps", type=float, default=1e-3)
    b.add_argument("--device", default="cuda", choices=("cuda",))
    b.add_argument("--out", default="-")
    a = ap.parse_args(argv)

    from .api import SolverConfig
    from .benchrun import BenchJob, bench_csv, run_bench
    from .instances import GenSpec, shape_for_nnz

    cfg = SolverConfig(eps_prim=a.eps, eps_dual=a.eps, eps_gap=a.eps)
    jobs = []
    for size in (float(s) for s in a.nnz.split(",")):
        for dens in (float(s) for s in a.density.split(",")):
            m, n = shape_for_nnz(int(size), dens, a.cone)
            jobs.append(BenchJob(len(jobs), GenSpec(m, n, dens, a.cone, seed=a.seed + len(jobs)), cfg))
    text = bench_csv(run_bench(jobs), extra=True)
    if a.out == "-":
        sys.stdout.write(text)
    else:
        with open(a.out, "w", encoding="utf-8") as f:
            f.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
