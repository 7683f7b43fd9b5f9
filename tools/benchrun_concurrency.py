"""Wall time of run_bench over 16 mid-size jobs (~1e5 nonzeros) at 1, 2, 4 and 8 workers."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.benchrun import BenchJob, run_bench
    from paper_2203_05027_b200.instances import GenSpec, shape_for_nnz

    m, n = shape_for_nnz(100_000, 0.01)
    cfg = SolverConfig(eps_prim=1e-3, eps_dual=1e-3, eps_gap=1e-3)
    jobs = [BenchJob(i, GenSpec(m, n, 0.01, "lp", seed=i), cfg) for i in range(16)]
    run_bench(jobs[:2], workers=2)   # warm-up
    for w in (1, 2, 4, 8):
        t0 = time.perf_counter()
        rows = run_bench(jobs, workers=w)
        dt = time.perf_counter() - t0
        its = sum(r["iters"] for r in rows)
        print(f"workers={w}: {dt:.2f} s for {len(rows)} jobs, {its} iterations ({its / dt:.0f} it/s)")


if __name__ == "__main__":
    main()
