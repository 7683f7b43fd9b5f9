"""One batched-kernel launch for profiling: 148 copies of a C4 problem, 5000 forced iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve_batch

    p = generate(GenSpec(100, 200, 0.05, "lp", seed=0))
    tim = {}
    solve_batch([p] * 148, SolverConfig(max_iters=5000, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0), trace=False,
                timing=tim)
    print(f"{tim['kernel_ms'] * 1e3 / 5000:.2f} us per iteration")


if __name__ == "__main__":
    main()
