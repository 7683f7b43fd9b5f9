"""bench.py's N>1 path (run_strong) on CPU: gloo, world 2, the numpy rank backends.

The driver launches ``bench.py --gpus N`` under torchrun for its scaling curve; this
runs that exact function (layout choice, warm-up, timed loop, max-over-ranks timing,
time-to-tolerance and the solve_distributed e2e) with the test backends of
test_sharded.py in place of the CUDA ones, and checks its line against the oracle.
"""

import contextlib
import json
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from test_sharded import NumpyColBackend, NumpyRankBackend, _free_port

from paper_2203_05027_b200 import SolverConfig, cfgen


def _worker(rank, world, port, shape, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench

        m, n, dens, kind = shape
        p = cfgen.generate_host(m, n, dens, kind, 0).problem()
        args = bench.parse_args(["--steps", "50", "--warmup", "3", "--gpus", str(world), "--eps", "1e-3"])
        spec = dict(bench.CONFIGS["c2"], m=m, n=n, density=dens, cone_kind=kind)
        with open(out_path if rank == 0 else os.devnull, "w") as f, contextlib.redirect_stdout(f):
            bench.run_strong(args, spec, rank, world, 0,
                             factories={"rows": NumpyRankBackend, "cols": NumpyColBackend}, problem=p)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape,mode", [((40, 100, 0.1, "lp"), "cols"), ((150, 80, 0.05, "lp"), "rows")])
def test_run_strong_world2(tmp_path, shape, mode):
    out = str(tmp_path / "line.json")
    mp.start_processes(_worker, args=(2, _free_port(), shape, out), nprocs=2, join=True, start_method="spawn")
    line = json.loads(open(out).read().strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong" and line["steps"] == 50
    assert line["config"]["parallelism"].startswith(f"{mode}-sharded x2")
    assert line["value"] > 0 and line["ms_per_step"] > 0
    m, n, dens, kind = shape
    p = cfgen.generate_host(m, n, dens, kind, 0).problem()
    cfg = SolverConfig(eps_prim=1e-3, eps_dual=1e-3, eps_gap=1e-3)
    _, _, tr, _ = oracle.solve(p, cfg)
    assert line["time_to_tol"]["iters"] == tr[-1]["iter"] and line["time_to_tol"]["status"] == tr[-1]["status"]
    assert line["e2e"]["iters"] == tr[-1]["iter"] and line["e2e"]["status"] == tr[-1]["status"]
    np.testing.assert_allclose(line["time_to_tol"]["pobj"], tr[-1]["pobj"], rtol=1e-9, atol=1e-9)
    assert line["iteration_roofline"]["nvlink_bytes_per_rank_per_iteration"] > 0
