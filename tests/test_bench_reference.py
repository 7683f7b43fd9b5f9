"""bench.py --impl reference runs on CPU only and never loads libcfb200.

C4: the batch metric (problem-iterations/s, the unit of our C4 arm) from the reference's own
run_bench process pool (bench.py:96-106 of the reference; the oracle port without baseline/_ref).
C1: the full reference solve to 1e-4 on the reference's own instance (11,375 iterations)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_batch_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c4", "--cpu-budget", "2"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["unit"] == "problem-iterations/s"
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    cpu = line["cpu_baseline"]
    assert cpu["kind"] in ("reference", "port") and cpu["cores"] == (os.cpu_count() or 1)
    assert cpu["value"] == line["value"]
    assert line["native_so_loaded"] == []          # the reference arm never maps libcfb200
    assert line["config"]["problems"] == 4096


def test_reference_arm_c1_full_solve():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "iterations/s"
    assert line["time_to_tol"]["iters"] == 11375 and line["time_to_tol"]["status"] == "solved"
    assert abs(line["time_to_tol"]["pobj"] - 220.7838450224) < 1e-6
    assert line["cpu_baseline"]["cores"] == 1 and line["cpu_baseline"]["host_cores"] == (os.cpu_count() or 1)
    assert line["native_so_loaded"] == []
    assert line["e2e"]["value"] == line["value"]
