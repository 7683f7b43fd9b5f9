"""GPU benchmark sweep with the reference's bench API (conefree/bench.py).

Same jobs, same rows, same CSV as the reference's ``run_bench``:
``BENCH_COLUMNS`` (bench.py:22-38) unchanged, every deterministic column equal
to what the reference produces for the job (instances come from the
bit-identical generator in ``instances.py``; solves from ``solve`` /
``solve_batch``, which match ``conefree.solve`` iteration for iteration).
``time_ms`` is wall time around the solve as in bench.py:60-62; for jobs
solved together by ``solve_batch`` it is the batch time divided evenly.

Where the reference spreads jobs over a process pool (bench.py:96-106), this
module runs small jobs as one batched launch (one CTA per problem) and larger
ones a few at a time, each with its own plan and CUDA stream. ``EXTRA_COLUMNS`` adds iterations/s, the
solve's HBM GB/s under the algorithmic byte count and its
fraction of the measured peak; ``bench_csv(rows, extra=True)`` prints them.
"""

from __future__ import annotations

import json
import os
import time
from dataclasses import dataclass

from .api import SolverConfig, solve, solve_batch
from .instances import GenSpec, generate, shape_for_nnz

__all__ = ["BENCH_COLUMNS", "EXTRA_COLUMNS", "BenchJob", "shape_for_nnz", "run_job", "run_bench", "bench_csv"]

BENCH_COLUMNS = (
    "instance_id",
    "m",
    "n",
    "nnz",
    "density",
    "cone_kind",
    "mu",
    "term_mode",
    "iters",
    "time_ms",
    "prim_res_2",
    "dual_res_2",
    "gap",
    "cone_gap",
    "status",
)
EXTRA_COLUMNS = ("iters_per_s", "hbm_gbs", "roofline_frac")

# problems up to this many nonzeros are batched (one CTA each) by run_bench
BATCH_MAX_NNZ = 20_000


@dataclass(frozen=True)
class BenchJob:
    instance_id: int
    gen: GenSpec
    cfg: SolverConfig


def _hbm_peak() -> float:
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(path))["hbm_gbs"])
    except Exception:
        return 6562.6


def _row(job: BenchJob, problem, rep, elapsed_ms: float) -> dict:
    m, n, o = job.gen.m, job.gen.n, problem.A.nnz
    row = {
        "instance_id": job.instance_id,
        "m": m,
        "n": n,
        "nnz": o,
        "density": job.gen.density,
        "cone_kind": job.gen.cone_kind,
        "mu": job.cfg.mu,
        "term_mode": job.cfg.term_mode,
        "iters": rep.iter,
        "time_ms": elapsed_ms,
        "prim_res_2": rep.prim_res_2,
        "dual_res_2": rep.dual_res_2,
        "gap": rep.gap,
        "cone_gap": rep.cone_gap,
        "status": rep.status,
    }
    sec = max(elapsed_ms, 1e-9) / 1e3
    gbs = rep.iter * (24 * o + 44 * m + 68 * n) / sec / 1e9
    row.update({"iters_per_s": rep.iter / sec, "hbm_gbs": gbs, "roofline_frac": gbs / _hbm_peak()})
    return row


def run_job(job: BenchJob) -> dict:
    """Generate and solve one instance on the GPU; the reference's row (bench.py:58-81)."""
    problem = generate(job.gen)
    start = time.perf_counter()
    result = solve(problem, job.cfg)
    elapsed_ms = (time.perf_counter() - start) * 1e3
    return _row(job, problem, result.report, elapsed_ms)


def run_bench(jobs, workers: int | None = None, batch_max_nnz: int = BATCH_MAX_NNZ) -> list:
    """Run all jobs and return rows sorted by instance_id (bench.py:96-106).

    Jobs with at most ``batch_max_nnz`` nonzeros that share a SolverConfig are
    solved together by ``solve_batch`` (one CTA per problem). Larger jobs run
    ``workers`` at a time (default ``CONEFREE_THREADS`` or 8), each in its own
    host thread with its own plan and CUDA stream: a mid-size solve leaves most
    of the GPU idle, so concurrent solves fill it (the reference spreads jobs
    over a process pool for the same reason; 16 jobs of 1e5 nonzeros: 3.9x the serial
    throughput at 8 workers, tools/benchrun_concurrency.py). Every row equals the serial run's."""
    from concurrent.futures import ThreadPoolExecutor

    if workers is None:
        env = os.environ.get("CONEFREE_THREADS")
        workers = int(env) if env else 8
    workers = max(1, int(workers))
    jobs = list(jobs)
    rows = []
    small: dict = {}
    large = []
    for job in jobs:
        if job.gen.nnz <= batch_max_nnz:
            small.setdefault(job.cfg, []).append(job)
        else:
            large.append(job)
    for cfg, group in small.items():
        problems = [generate(j.gen) for j in group]
        start = time.perf_counter()
        try:
            results = solve_batch(problems, cfg, trace=False)
        except ValueError:
            # a problem that does not fit one CTA: solve it like a large job
            large.extend(group)
            continue
        per_ms = (time.perf_counter() - start) * 1e3 / len(group)
        rows.extend(_row(j, p, r.report, per_ms) for j, p, r in zip(group, problems, results))
    if workers == 1 or len(large) <= 1:
        rows.extend(run_job(j) for j in large)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            rows.extend(pool.map(run_job, large))
    return sorted(rows, key=lambda r: r["instance_id"])


def _cell(value) -> str:
    if isinstance(value, float):
        return repr(value)
    return str(value)


def bench_csv(rows, extra: bool = False) -> str:
    """The reference's CSV (bench.py:115-119); extra=True appends EXTRA_COLUMNS."""
    cols = BENCH_COLUMNS + (EXTRA_COLUMNS if extra else ())
    lines = [",".join(cols)]
    for row in rows:
        lines.append(",".join(_cell(row[c]) for c in cols))
    return "\n".join(lines) + "\n"
