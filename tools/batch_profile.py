"""Host-side profile of solve_batch on the C4 batch (cProfile, top functions by cumulative time)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve_batch

    probs = [generate(GenSpec(100, 200, 0.05, "lp", seed=s)) for s in range(4096)]
    cfg = SolverConfig(eps_prim=1e-4, eps_dual=1e-4, eps_gap=1e-4)
    solve_batch(probs[:64], SolverConfig(max_iters=100), trace=False)
    tim = {}
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    solve_batch(probs, cfg, trace=False, timing=tim)
    pr.disable()
    print(f"total {time.perf_counter() - t0:.3f} s, kernel {tim['kernel_ms'] / 1e3:.3f} s")
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()
