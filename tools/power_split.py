"""Clock and power per pass under sustained load (C2): full iterations, column passes only,
row passes only, each for a few seconds with nvidia-smi sampled meanwhile.

    python tools/power_split.py [seconds]
"""
import ctypes
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def sample(fn, seconds):
    import torch

    log = "/tmp/power_split_smi.csv"
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "100"], stdout=open(log, "w"))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    n = 0
    e0.record()
    while time.time() - t0 < seconds:
        n += fn()
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    smi.terminate()
    smi.wait()
    rows = [l.split(",") for l in open(log) if l.strip()]
    clk = [float(r[0]) for r in rows[5:]]
    pw = [float(r[1]) for r in rows[5:]]
    return e0.elapsed_time(e1) / n, statistics.median(clk), statistics.median(pw), max(pw)


def main():
    import torch

    from bench import CONFIGS, device_instance
    from paper_2203_05027_b200 import _lib

    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 6.0
    st = torch.cuda.current_stream()
    inst = device_instance(CONFIGS["c2"], 0, st.cuda_stream)
    plan = inst.plan
    plan.set_state(1.0, None, export=False)
    lib = _lib.lib()
    h = plan.handle

    def full():
        _lib.check(lib.cf_plan_iterate(h, 1.0, 200))
        return 200

    def col():
        for _ in range(200):
            _lib.check(lib.cf_plan_col_step(h, 1.0))
        return 200

    def row():
        for _ in range(200):
            _lib.check(lib.cf_plan_row_step(h, 1.0, 0))
        return 200

    import torch as _t

    hv = _t.zeros(inst.m, dtype=_t.float64, device="cuda")
    xv = _t.zeros(inst.n, dtype=_t.float64, device="cuda")

    def spmv_t():   # A^T h alone: the column pass's sums without its epilogue
        for _ in range(200):
            _lib.check(lib.cf_apply_At_async(h, ctypes.c_void_p(hv.data_ptr()), ctypes.c_void_p(xv.data_ptr())))
        return 200

    full()
    torch.cuda.synchronize()
    for name, fn in (("iteration", full), ("column pass", col), ("A^T h only", spmv_t), ("row pass", row),
                     ("iteration", full)):
        ms, clk, pw, pmax = sample(fn, secs)
        print(f"{name:12s} {ms:.4f} ms  sm clock median {clk:.0f} MHz  power median {pw:.0f} W (max {pmax:.0f})",
              flush=True)


if __name__ == "__main__":
    main()
