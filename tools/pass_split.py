"""Per-pass device time (row / column pass) at one size, C2 structure: python tools/pass_split.py 1000000"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(o):
    import torch

    from paper_2203_05027_b200 import SolverConfig
    from paper_2203_05027_b200.devgen import generate_device
    from paper_2203_05027_b200.engine import config_struct

    st = torch.cuda.current_stream()
    m = o // 20
    inst = generate_device(m, 2 * m, 20.0 / (2 * m), "lp", seed=1, stream=st.cuda_stream)
    plan = inst.plan
    cfg = config_struct(SolverConfig(max_iters=400, eps_prim=0.0, eps_dual=0.0, eps_gap=0.0), (1.0, 1.0), (1.0, 1.0))
    plan.set_state(1.0, None, export=False)
    plan.run(cfg, want_x=False)
    plan.set_state(1.0, None, export=False)
    plan.set_profiling(True)
    plan.run(cfg, want_x=False)
    t = plan.last_timing()
    print(f"o={o}: row {t['row_pass_ms'] * 1e3 / 400:.2f} us, col {t['col_pass_ms'] * 1e3 / 400:.2f} us, "
          f"loop {t['loop_ms'] * 1e3 / 400:.2f} us/iteration, info {plan.info()}")


if __name__ == "__main__":
    main(int(float(sys.argv[1])))
