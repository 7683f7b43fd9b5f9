"""Per-iteration latency of the batched kernel: one problem (one CTA) forced to max_iters."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from paper_2203_05027_b200 import GenSpec, SolverConfig, generate, solve_batch

    p = generate(GenSpec(100, 200, 0.05, "lp", seed=0))
    for P in (1, 148, 444, 888):
        cfg = SolverConfig(max_iters=20000, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0)
        tim = {}
        solve_batch([p] * P, cfg, trace=False, timing=tim)
        print(f"P={P}: kernel {tim['kernel_ms']:.1f} ms -> {tim['kernel_ms'] * 1e3 / 20000:.2f} us per iteration "
              f"({P * 20000 / tim['kernel_ms'] / 1e3:.1f} M problem-it/s)")


if __name__ == "__main__":
    main()
