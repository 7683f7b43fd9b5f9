"""Per-iteration time across problem sizes (C2 structure: 20 nnz/row, n = 2m), no per-pass events.

    python tools/prof_sizes.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2203_05027_b200.devgen import generate_device

    st = torch.cuda.current_stream()
    for o in (20_000, 100_000, 1_000_000, 3_000_000, 10_000_000, 30_000_000, 100_000_000):
        m = o // 20
        n = 2 * m
        inst = generate_device(m, n, 20.0 / n, "lp", seed=1, stream=st.cuda_stream)
        plan = inst.plan
        plan.set_state(1.0, None, export=False)
        iters = 400 if o <= 3_000_000 else 100
        plan.iterate(1.0, 20)
        torch.cuda.synchronize()
        plan.iterate(1.0, iters)
        t = plan.last_timing()
        info = plan.info()
        print(f"o={o:>11,d} m={m:>9,d} n={n:>10,d} row_tiles={info['row_tiles']:>6d} col_tiles={info['col_tiles']:>6d}: "
              f"{t['loop_ms'] * 1e3 / iters:8.1f} us/iteration")
        plan.close()
        del inst
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
