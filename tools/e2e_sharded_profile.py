"""Where the host time of solve_distributed goes (C2, world 1, column layout)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    import bench
    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.api import norms
    from paper_2203_05027_b200.devgen import to_host_problem
    from paper_2203_05027_b200.problem import cone_sizes_array
    from paper_2203_05027_b200.sharded import CudaColBackend, column_cuts, local_columns, run_col_sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29541")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    inst = bench.device_instance(bench.CONFIGS["c2"], 0, torch.cuda.current_stream().cuda_stream)
    inst.plan.close()
    p = to_host_problem(inst)
    del inst
    torch.cuda.empty_cache()
    cfg = SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)
    for rep in range(2):
        t = {}
        t0 = time.perf_counter()
        cuts = column_cuts(cone_sizes_array(p.cones), int(p.A.num_cols), 1)
        t["cuts"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        lp = local_columns(p, cuts[0], cuts[1])
        t["local_columns"] = time.perf_counter() - t1
        t1 = time.perf_counter()
        be = CudaColBackend(lp)
        torch.cuda.synchronize()
        t["backend (H2D + setup)"] = time.perf_counter() - t1
        t1 = time.perf_counter()
        bn, cn = norms(p.b), norms(p.c)
        t["norms"] = time.perf_counter() - t1
        t1 = time.perf_counter()
        tim = {}
        res = run_col_sharded(be, cuts, cfg if rep else SolverConfig(max_iters=25), bn, cn, timing=tim)
        t["loop + gather"] = time.perf_counter() - t1
        t["loop device ms"] = tim.get("loop_ms")
        t1 = time.perf_counter()
        be.close()
        t["close"] = time.perf_counter() - t1
        t["total"] = time.perf_counter() - t0
        print(rep, res.report.iter, {k: round(v, 3) if isinstance(v, float) else v for k, v in t.items()}, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
